#!/bin/bash
# march_kernel: parity (default build), RS=1 (reconstruction over K+1 warps) vs RS=0, phase profile.
mkdir -p gpurun_out; : > gpurun_out/march2.log
timeout 900 python -m pytest tests -q -m gpu -x >> gpurun_out/march2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/march2.log
for rep in 1 2; do
for rs in 1 0; do
for cs in 8 16; do
echo "rs=$rs cs=$cs $(MGP_MARCH_RS=$rs MGP_MARCH_CS=$cs timeout 300 python tools/kernel_times.py c2 c3 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print(d['c2_march_us_per_step'], d['c3_march_us_per_step'])")" >> gpurun_out/march2.log
done; done; done
for rs in 1 0; do
echo "prof rs=$rs c2 cs=8 $(MGP_MARCH_RS=$rs MGP_LIB_PATH=tools/exp/lib_trace.so MGP_MARCH_CS=8 timeout 120 python tools/march_prof.py c2 2>&1 | tail -1)" >> gpurun_out/march2.log
done
