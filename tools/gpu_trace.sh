#!/bin/bash
mkdir -p gpurun_out
for cs in 1 4 8; do echo "== cs=$cs" >> gpurun_out/trace.log; MGP_LIB_PATH=tools/exp/lib_trace.so MGP_MARCH_CS=$cs timeout 120 python tools/trace_march.py c2 >> gpurun_out/trace.log 2>&1; done
