#!/bin/bash
# march_kernel A/B (tools/exp/libmgrit_phi_old.so = previous build) + GPU suite.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do
for lib in old new; do
  if [ $lib = old ]; then export MGP_LIB_PATH=$PWD/tools/exp/libmgrit_phi_old.so; else unset MGP_LIB_PATH; fi
  echo "$lib $(timeout 300 python tools/kernel_times.py c2 c3 | tr -d '\n ')" >> gpurun_out/march_ab.log
  echo "$lib $(timeout 300 python tools/iter_times.py c2 | python -c 'import json,sys; d=json.load(sys.stdin); print(d["c2"]["iteration_ms"])')" >> gpurun_out/march_ab.log
done; done
unset MGP_LIB_PATH
