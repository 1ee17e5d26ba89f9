mkdir -p gpurun_out; : > gpurun_out/e2e.log
python - >> gpurun_out/e2e.log 2>&1 <<'PY'
import torch, time
x = torch.empty(16 * 2**20 // 8, dtype=torch.float64, device="cuda")
h = torch.empty_like(x, device="cpu").pin_memory()
for name, f in (("d2h", lambda: h.copy_(x, non_blocking=True)), ("h2d", lambda: x.copy_(h, non_blocking=True))):
    f(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20): f()
    b.record(); torch.cuda.synchronize()
    print(name, "GB/s", 20 * x.numel() * 8 / (a.elapsed_time(b) * 1e-3) / 1e9)
PY
for p in 1 2 4 8 16; do
for g in 0 1; do
echo "pieces=$p graph=$g $(MGP_E2E_PIECES=$p MGP_E2E_GRAPH=$g timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['e2e']['value'], d['value'])")" >> gpurun_out/e2e.log
done; done
