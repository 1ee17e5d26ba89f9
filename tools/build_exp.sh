#!/bin/bash
# quick experiment build: tools/build_exp.sh NAME [extra nvcc flags]  -> tools/exp/NAME.so
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true \
  -prec-sqrt=true -diag-suppress 128 -Xcompiler -fPIC -shared -DMGP_QUICK -Xptxas -v "$@" \
  -I include -o tools/exp/$name.so paper_2104_09404_b200/csrc/mgrit_phi.cu > tools/exp/$name.ptxas 2>&1
echo "$name rc=$?"
grep -A1 'sweep_kernelILi2ELi0ELi0ELi4ELi128ELi1E' tools/exp/$name.ptxas | grep -o '[0-9]* bytes spill stores'
