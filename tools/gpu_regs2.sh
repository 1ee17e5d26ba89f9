#!/bin/bash
# production builds: 128 vs 96 registers (fcf_kernel + sweep_kernel), probe + bench.
mkdir -p gpurun_out; : > gpurun_out/regs2.log
for rep in 1 2; do
for lib in paper_2104_09404_b200/libmgrit_phi.so tools/exp/lib_prod_r96.so; do
echo "$lib $(MGP_LIB_PATH=$lib timeout 300 python tools/fcf_probe.py 592 1024 2368 4736 2>&1 | tail -1)" >> gpurun_out/regs2.log
echo "$lib bench $(MGP_LIB_PATH=$lib timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['iteration_ms'])")" >> gpurun_out/regs2.log
echo "$lib kt $(MGP_LIB_PATH=$lib MGP_KT_NOMARCH=1 timeout 300 python tools/kernel_times.py c2 c3 2>&1 | tr -d '\n')" >> gpurun_out/regs2.log
done; done
