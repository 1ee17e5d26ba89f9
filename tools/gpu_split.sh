#!/bin/bash
# Split plan of the fused FCF relaxation: parity, probe over interval counts, bench A/B.
mkdir -p gpurun_out; : > gpurun_out/split.log
timeout 600 python -m pytest tests/test_gpu_fcf.py -q -m gpu -x >> gpurun_out/split.log 2>&1; echo "fcf tests rc=$?" >> gpurun_out/split.log
MGP_PROBE_SPLITS="148 296 444 800" timeout 300 python tools/fcf_probe.py 296 592 1024 1184 2368 4736 >> gpurun_out/split.log 2>&1
for sp in -1 0 -1 0; do
echo "split=$sp $(MGP_BENCH_SPLIT=$sp timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['frac'], d['e2e']['value'])")" >> gpurun_out/split.log
done
for p in 0 1; do
echo "split=0 pieces=$p $(MGP_E2E_PIECES=$p timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['e2e']['value'])")" >> gpurun_out/split.log
done
