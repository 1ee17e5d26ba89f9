#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/mprof.log
for cs in 4 8 16; do
echo "c2 cs=$cs $(MGP_LIB_PATH=tools/exp/lib_trace.so MGP_MARCH_CS=$cs timeout 120 python tools/march_prof.py c2 2>&1 | tail -1)" >> gpurun_out/mprof.log
done
echo "c3 cs=16 $(MGP_LIB_PATH=tools/exp/lib_trace.so MGP_MARCH_CS=16 timeout 120 python tools/march_prof.py c3 2>&1 | tail -1)" >> gpurun_out/mprof.log
