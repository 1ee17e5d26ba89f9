#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/march.log
for cs in 2 4 8 16; do
  echo "cs=$cs $(MGP_MARCH_CS=$cs timeout 120 python tools/kernel_times.py c2 c3 2>&1 | tr -d '\n ')" >> gpurun_out/march.log
done
