#!/bin/bash
# Full round check: smoke, gpu tests, default bench, reference arm, ncu launch list + full capture.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
$CMD > gpurun_out/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:fcf_kernel -s 1 -c 1 -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
timeout 600 python tools/iter_times.py c2 c3 c5 > gpurun_out/iter_times.json 2> gpurun_out/iter_times.err; echo "iter rc=$?" >> gpurun_out/iter_times.err
timeout 300 python tools/kernel_times.py c2 c3 > gpurun_out/kernel_times.json 2>&1
