#!/bin/bash
# ncu full captures of the sequential march (C2 coarse/serial march) and the
# C5 cluster sweep; refreshed iteration timings.
mkdir -p gpurun_out
timeout 300 python tools/kernel_times.py c2 > gpurun_out/kt_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:march_kernel -c 1 -o gpurun_out/prof_march python tools/kernel_times.py c2 > gpurun_out/ncu_march.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_march.log
MGP_KT_NOMARCH=1 MGP_KT_MAXCHUNKS=148 timeout 300 python tools/kernel_times.py c5 > gpurun_out/kt_c5_148.json 2>&1 && \
MGP_KT_NOMARCH=1 MGP_KT_MAXCHUNKS=148 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o gpurun_out/prof_c5 python tools/kernel_times.py c5 > gpurun_out/ncu_c5.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_c5.log
timeout 600 python tools/iter_times.py c2 c3 c5 > gpurun_out/iter_times.json 2> gpurun_out/iter_times.err
# summaries on the box; the reports themselves are too big to bring back together
for r in march c5; do
  python tools/ncu_summary.py gpurun_out/prof_$r.ncu-rep > gpurun_out/ncu_${r}_summary.json 2>&1
  python tools/ncu_src_summary.py gpurun_out/prof_$r.ncu-rep > gpurun_out/ncu_${r}_source.txt 2>&1
  ncu -i gpurun_out/prof_$r.ncu-rep --page details --csv > gpurun_out/ncu_${r}_details.csv 2>&1
  rm -f gpurun_out/prof_$r.ncu-rep
done
