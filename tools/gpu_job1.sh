mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
: > gpurun_out/wave.log
for r in 4 8; do MGP_RUN=$r timeout 120 python tools/wave_probe.py >> gpurun_out/wave.log 2>&1; done
MGP_KT_NOMARCH=1 MGP_LIB_PATH=tools/exp/v8.so MGP_MAXREG=96 timeout 120 python tools/wave_probe.py >> gpurun_out/wave.log 2>&1
MGP_KT_NOMARCH=1 MGP_LIB_PATH=tools/exp/v8.so MGP_MAXREG=96 MGP_RUN=8 timeout 120 python tools/wave_probe.py >> gpurun_out/wave.log 2>&1
MGP_KT_NOMARCH=1 MGP_LIB_PATH=tools/exp/v8.so MGP_MAXREG=112 timeout 120 python tools/wave_probe.py >> gpurun_out/wave.log 2>&1
