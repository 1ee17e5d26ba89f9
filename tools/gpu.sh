#!/bin/bash
# One parameterised launcher for gpurun calls; every log goes to gpurun_out/.
#
#   tools/gpu.sh check [pytest-args]     smoke + `pytest -m gpu` + short bench
#   tools/gpu.sh round                   smoke, gpu tests, default bench, reference
#                                        arm, ncu launch list + full capture of
#                                        fcf_kernel, iteration / kernel times
#   tools/gpu.sh bench [bench args]      one bench.py run
#   tools/gpu.sh ncu TAG REGEX SKIP CMD  plain run of CMD, then one ncu --set full
#                                        capture of the SKIP-th launch matching REGEX
#   tools/gpu.sh launches TAG CMD        plain run of CMD, then its ncu launch list
#   tools/gpu.sh py SCRIPT [args]        any python script (timings, probes)
#
# e.g. gpurun --timeout 1800 -- 'bash tools/gpu.sh check -k full'
set -u
mkdir -p gpurun_out
what=${1:-check}; shift || true
case "$what" in
check)
    nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
    echo "smoke rc=$?" >> gpurun_out/smoke.log
    timeout 3000 python -m pytest tests -q -m gpu "$@" > gpurun_out/pytest_gpu.log 2>&1
    echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
    timeout 900 python bench.py --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/bench.log 2>&1
    echo "bench rc=$?" >> gpurun_out/bench.log
    tail -n 3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log gpurun_out/bench.log ;;
round)
    timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
    echo "smoke rc=$?" >> gpurun_out/smoke.log
    timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
    echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
    timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
    timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
    echo "ref rc=$?" >> gpurun_out/bench_ref.log
    CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline"
    $CMD > gpurun_out/bench_plain.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:fcf_kernel -s 1 -c 1 \
        -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
    echo "ncu rc=$?" >> gpurun_out/ncu_full.log ;;
bench)
    timeout 900 python bench.py "$@" > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
    tail -n 2 gpurun_out/bench.log ;;
ncu)
    tag=$1; regex=$2; skip=$3; shift 3
    "$@" > gpurun_out/plain_$tag.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k "regex:$regex" -s "$skip" -c 1 \
        -o gpurun_out/prof_$tag "$@" > gpurun_out/ncu_$tag.log 2>&1
    echo "ncu rc=$?" >> gpurun_out/ncu_$tag.log; tail -n 3 gpurun_out/ncu_$tag.log ;;
launches)
    tag=$1; shift
    "$@" > gpurun_out/plain_$tag.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches_$tag.csv "$@" > gpurun_out/ncu_launch_$tag.log 2>&1
    echo "ncu rc=$?" >> gpurun_out/ncu_launch_$tag.log ;;
py)
    script=$1; shift
    base=$(basename "$script" .py)
    timeout 1800 python "$script" "$@" > gpurun_out/$base.out 2> gpurun_out/$base.err
    echo "rc=$?" >> gpurun_out/$base.err; tail -n 5 gpurun_out/$base.out gpurun_out/$base.err ;;
*)
    echo "unknown mode $what"; exit 2 ;;
esac
