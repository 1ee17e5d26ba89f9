#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/exp.log
for run in 4 8; do for reg in 0 112 104 96 80; do
  echo "run=$run reg=$reg $(MGP_LIB_PATH=tools/exp/lib_exp.so MGP_RUN=$run MGP_MAXREG=$reg timeout 120 python tools/kernel_times.py c2 c3 2>&1 | tr -d '\n ')" >> gpurun_out/exp.log
done; done
