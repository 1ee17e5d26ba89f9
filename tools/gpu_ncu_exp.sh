#!/bin/bash
# ncu --set full of one C2 fused F+C sweep launch of tools/exp/$1.so
mkdir -p gpurun_out
MGP_LIB_PATH=tools/exp/$1.so timeout 120 python tools/kernel_times.py c2 > gpurun_out/kt_$1.log 2>&1
MGP_LIB_PATH=tools/exp/$1.so timeout 600 ncu --set full --clock-control none \
  -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/exp_$1 python tools/kernel_times.py c2 > gpurun_out/ncu_$1.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_$1.log
