#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/lat.log
./tools/fp64_latency >> gpurun_out/lat.log 2>&1
for p in 0 4 0 4 0 4; do
echo "pieces=$p $(MGP_E2E_PIECES=$p timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['e2e']['value'], d['iteration_ms'])")" >> gpurun_out/lat.log
done
