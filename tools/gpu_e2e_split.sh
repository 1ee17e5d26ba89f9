mkdir -p gpurun_out; : > gpurun_out/e2e_split.log
for r in 1 2; do for sp in 0 -1 1184; do
echo "split=$sp $(MGP_BENCH_SPLIT=$sp timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | grep '^{' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['e2e']['value'], d['value'])")" >> gpurun_out/e2e_split.log
done; done
for sg in 1 2; do
echo "segment=$sg $(MGP_BENCH_SEGMENT=$sg timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | grep '^{' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['e2e']['value'], d['value'])")" >> gpurun_out/e2e_split.log
done
