#!/bin/bash
: > gpurun_out/e2e.log
timeout 300 python -m pytest tests/test_gpu_mgrit.py -q -m gpu -x -k relax_to_host > gpurun_out/pytest_e2e.log 2>&1; echo rc=$? >> gpurun_out/pytest_e2e.log
for g in 0 1; do for p in 2 3; do
  echo "graph=$g pieces=$p $(MGP_E2E_GRAPH=$g MGP_E2E_PIECES=$p timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | python -c 'import json,sys; l=json.loads(sys.stdin.readline()); print(l["value"], l["e2e"]["value"])')" >> gpurun_out/e2e.log
done; done
