#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/march.log
for cs in 1 2 4 8 16; do
  echo "cs=$cs $(MGP_MARCH_CS=$cs timeout 120 python tools/kernel_times.py c2 c3 2>&1 | tr -d '\n ')" >> gpurun_out/march.log
done
