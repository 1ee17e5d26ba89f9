#!/bin/bash
# register-cap variants of the quick build (release codegen): fused FCF and sweeps
mkdir -p gpurun_out; : > gpurun_out/regs3.log
for rep in 1 2; do for r in 128 168 96; do
  echo "regs=$r fcf $(MGP_LIB_PATH=$PWD/tools/exp/q$r.so timeout 300 python tools/fcf_probe.py 592 1024 2368 | tr -d '\n ')" >> gpurun_out/regs3.log
  echo "regs=$r kt $(MGP_LIB_PATH=$PWD/tools/exp/q$r.so MGP_KT_NOMARCH=1 timeout 300 python tools/kernel_times.py c2 c3 | tr -d '\n ')" >> gpurun_out/regs3.log
done; done
