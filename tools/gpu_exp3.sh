#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/exp3.log
for v in s0 s1; do
  echo "$v $(MGP_LIB_PATH=tools/exp/lib_$v.so timeout 120 python tools/kernel_times.py c2 c3 2>&1 | tr -d '\n ')" >> gpurun_out/exp3.log
done
MGP_LIB_PATH=tools/exp/lib_s1.so timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_s1.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_s1.log
