#!/bin/bash
# ordered zero-copy chain-start loads: parity, e2e probe, bench e2e by window
mkdir -p gpurun_out; : > gpurun_out/ordered.log
timeout 900 python -m pytest tests/test_gpu_fcf.py -q -m gpu -x > gpurun_out/pytest_fcf.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fcf.log
for r in 1 2; do for w in 0 96 128 192 256 384; do
  echo "window=$w $(MGP_FCF_ORDERED=$w timeout 300 python tools/e2e_probe.py 2>&1 | head -1)" >> gpurun_out/ordered.log
  echo "window=$w bench $(MGP_FCF_ORDERED=$w timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | grep '^{' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['e2e']['value'], d['value'])")" >> gpurun_out/ordered.log
done; done
