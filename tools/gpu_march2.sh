#!/bin/bash
# march_kernel: parity (default build), plain vs split cluster barrier per-step times.
mkdir -p gpurun_out; : > gpurun_out/march2.log
timeout 900 python -m pytest tests -q -m gpu -x >> gpurun_out/march2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/march2.log
MGP_LIB_PATH=tools/exp/lib_split.so timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_mgrit.py -q -m gpu -x >> gpurun_out/march2.log 2>&1; echo "split pytest rc=$?" >> gpurun_out/march2.log
for rep in 1 2; do
for lib in paper_2104_09404_b200/libmgrit_phi.so tools/exp/lib_split.so; do
for cs in 8 16; do
echo "$lib cs=$cs $(MGP_LIB_PATH=$lib MGP_MARCH_CS=$cs timeout 300 python tools/kernel_times.py c2 c3 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print(d['c2_march_us_per_step'], d['c3_march_us_per_step'])")" >> gpurun_out/march2.log
done; done; done
