#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/march.log
for cs in 4 8 16; do
  echo "cs=$cs $(MGP_MARCH_CS=$cs timeout 60 python tools/kernel_times.py c2 c3 2>&1 | tr -d '\n ' | cut -c1-400)" >> gpurun_out/march.log
done
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
