#!/bin/bash
# march parity suite + fcf register-budget experiment (fast builds of the same source).
mkdir -p gpurun_out; : > gpurun_out/regs.log
timeout 900 python -m pytest tests -q -m gpu -x >> gpurun_out/regs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/regs.log
for rep in 1 2; do
for lib in lib_r128 lib_r96 lib_r80; do
echo "$lib $(MGP_LIB_PATH=tools/exp/$lib.so timeout 300 python tools/fcf_probe.py 592 1024 2368 2>&1 | tail -1)" >> gpurun_out/regs.log
done; done
