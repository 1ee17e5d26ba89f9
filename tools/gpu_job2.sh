mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fcf.py -q -m gpu -x > gpurun_out/pytest_fcf.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fcf.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
