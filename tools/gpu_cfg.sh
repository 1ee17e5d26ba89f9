#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x > gpurun_out/pytest_cfg.log 2>&1; echo "cfg rc=$?" >> gpurun_out/pytest_cfg.log
