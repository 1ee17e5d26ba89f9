#!/bin/bash
mkdir -p gpurun_out
for run in 4 8; do for reg in 128 96 80 64; do
  echo "run=$run reg=$reg $(MGP_RUN=$run MGP_MAXREG=$reg timeout 120 python tools/kernel_times.py c2 c3 2>&1 | tr -d '\n ')" >> gpurun_out/regsweep.log
done; done
