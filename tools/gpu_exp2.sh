#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/exp2.log
for v in u1 u2; do for run in 4 8; do
  echo "$v run=$run $(MGP_LIB_PATH=tools/exp/lib_$v.so MGP_RUN=$run timeout 120 python tools/kernel_times.py c2 c3 2>&1 | tr -d '\n ')" >> gpurun_out/exp2.log
done; done
