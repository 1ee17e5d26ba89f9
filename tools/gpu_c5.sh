#!/bin/bash
# C5 cluster-path A/B: old library (tools/exp/libmgrit_phi_old.so) vs current,
# cluster residency probe, cluster parity tests.
mkdir -p gpurun_out
./tools/exp/cluster_occupancy > gpurun_out/cluster_occupancy.txt 2>&1
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for lib in old new; do
  if [ $lib = old ]; then export MGP_LIB_PATH=$PWD/tools/exp/libmgrit_phi_old.so; else unset MGP_LIB_PATH; fi
  MGP_KT_NOMARCH=1 MGP_KT_MAXCHUNKS=1184 timeout 300 python tools/kernel_times.py c5 c3 > gpurun_out/kt_c5_$lib.json 2>&1
  timeout 300 python tools/iter_times.py c5 > gpurun_out/iter_c5_$lib.json 2>&1
done
unset MGP_LIB_PATH
