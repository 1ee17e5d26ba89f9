#!/bin/bash
# full GPU parity suite, then BASELINE config 4 in full (192 cases) and march timings.
mkdir -p gpurun_out; : > gpurun_out/c4.log
timeout 900 python -m pytest tests -q -m gpu -x >> gpurun_out/c4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/c4.log
timeout 900 python tools/c4_sweep.py > gpurun_out/c4_sweep.jsonl 2>> gpurun_out/c4.log; echo "c4 rc=$?" >> gpurun_out/c4.log
timeout 300 python tools/kernel_times.py c2 c3 >> gpurun_out/c4.log 2>&1
