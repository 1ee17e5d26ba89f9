#!/bin/bash
# fcf look-ahead prefetch: parity, e2e probe and bench (old = previous build)
mkdir -p gpurun_out; : > gpurun_out/pf.log
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for r in 1 2; do for lib in old new; do
  if [ $lib = old ]; then export MGP_LIB_PATH=$PWD/tools/exp/libmgrit_phi_old.so; else unset MGP_LIB_PATH; fi
  echo "== $lib" >> gpurun_out/pf.log
  timeout 300 python tools/e2e_probe.py >> gpurun_out/pf.log 2>&1
  echo "bench $(timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | grep '^{' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['e2e']['value'], d['value'])")" >> gpurun_out/pf.log
done; done
unset MGP_LIB_PATH
