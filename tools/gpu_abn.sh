#!/bin/bash
# A/B over experiment builds: tools/gpu_abn.sh v1 v2 ... (kernel_times c2 c3, fused F+C sweep)
mkdir -p gpurun_out
: > gpurun_out/abn.log
for i in 1 2; do
for v in "$@"; do
if [ "$v" = main ]; then lib=paper_2104_09404_b200/libmgrit_phi.so; else lib=tools/exp/$v.so; fi
echo "$v $(MGP_KT_NOMARCH=1 MGP_LIB_PATH=$lib timeout 120 python tools/kernel_times.py c2 c3 2>&1 | tr -d '\n ' | cut -c1-330)" >> gpurun_out/abn.log
done; done
