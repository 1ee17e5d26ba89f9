#!/bin/bash
mkdir -p gpurun_out; : > gpurun_out/mt.log
timeout 900 python -m pytest tests/test_gpu_march.py -q -m gpu -x >> gpurun_out/mt.log 2>&1; echo "pytest rc=$?" >> gpurun_out/mt.log
timeout 600 python tools/march_times.py >> gpurun_out/mt.log 2>&1
