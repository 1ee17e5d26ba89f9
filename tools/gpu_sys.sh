#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_euler.py tests/test_gpu_sw.py -q -x > gpurun_out/pytest_sys.log 2>&1; echo "sys rc=$?" >> gpurun_out/pytest_sys.log
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
