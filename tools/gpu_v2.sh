#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for r in 2 4 8; do MGP_RUN=$r timeout 300 python tools/kernel_times.py c2 c3 > gpurun_out/kt_run$r.log 2>&1; done
timeout 600 python bench.py --steps 10 --warmup 3 --cpu-seconds 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
