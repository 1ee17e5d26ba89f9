#!/bin/bash
# Stage trace of the sequential march (thread 0 of CTA 0, globaltimer) and
# per-step march times for several cluster sizes.
mkdir -p gpurun_out; : > gpurun_out/trace.log
for cs in 8 16; do echo "== c2 cs=$cs" >> gpurun_out/trace.log; MGP_LIB_PATH=tools/exp/lib_trace.so MGP_MARCH_CS=$cs timeout 120 python tools/trace_march.py c2 >> gpurun_out/trace.log 2>&1; done
echo "== c3 cs=16" >> gpurun_out/trace.log; MGP_LIB_PATH=tools/exp/lib_trace.so MGP_MARCH_CS=16 timeout 120 python tools/trace_march.py c3 >> gpurun_out/trace.log 2>&1
for cs in 4 8 16; do echo "cs=$cs $(MGP_MARCH_CS=$cs MGP_KT_NOFC=1 timeout 300 python tools/kernel_times.py c2 c3 2>&1 | tr -d '\n')" >> gpurun_out/trace.log; done
