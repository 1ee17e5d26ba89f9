#!/bin/bash
# A/B: main library vs tools/exp/$1.so on kernel_times (c2 c3); parity tests
# of the Burgers-WENO propagator on the variant ($2 = pytest -k filter)
mkdir -p gpurun_out
: > gpurun_out/ab.log
for i in 1 2; do
echo "main $(timeout 120 python tools/kernel_times.py c2 c3 2>&1 | tr -d '\n ' | cut -c1-330)" >> gpurun_out/ab.log
echo "$1 $(MGP_LIB_PATH=tools/exp/$1.so timeout 120 python tools/kernel_times.py c2 c3 2>&1 | tr -d '\n ' | cut -c1-330)" >> gpurun_out/ab.log
done
MGP_LIB_PATH=tools/exp/$1.so timeout 600 python -m pytest tests/test_gpu_phi.py tests/test_gpu_mgrit.py -q -m gpu -k "${2:-not nothing}" > gpurun_out/pytest_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ab.log
