mkdir -p gpurun_out; : > gpurun_out/e2e.log
timeout 300 python -m pytest tests/test_gpu_fcf.py -q -m gpu -k pieces >> gpurun_out/e2e.log 2>&1
for p in 0 4 0 4; do
echo "pieces=$p $(MGP_E2E_PIECES=$p timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['e2e']['value'], d['value'])")" >> gpurun_out/e2e.log
done
