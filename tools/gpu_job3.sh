mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/bench_seg.log
for S in 0 1 2 0 1 2; do
echo "S=$S $(MGP_BENCH_SEGMENT=$S timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['frac'], d['kernel_ms'], d['e2e']['value'], d['iteration_ms'])")" >> gpurun_out/bench_seg.log
done
