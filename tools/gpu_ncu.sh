#!/bin/bash
# usage: tools/gpu_ncu.sh <tag> ; profiles the c2 fused relaxation kernel
mkdir -p gpurun_out
CMD="python tools/kernel_times.py c2"
$CMD > gpurun_out/plain_$1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/prof_$1 $CMD > gpurun_out/ncu_$1.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$1.log
