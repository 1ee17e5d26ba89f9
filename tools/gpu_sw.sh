#!/bin/bash
# shallow-water kernel parity first, then the whole GPU suite
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sw.py -q -x > gpurun_out/pytest_sw.log 2>&1; echo "sw rc=$?" >> gpurun_out/pytest_sw.log
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
