#!/bin/bash
# Experiment build of the full library with extra flags (split compile, fast):
#   tools/build_var.sh NAME [nvcc flags...]  -> tools/exp/NAME.so
name=$1; shift
mkdir -p tools/exp
nvcc -split-compile=0 -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -prec-div=true -prec-sqrt=true -diag-suppress 128 -Xcompiler -fPIC -shared "$@" \
  -I include -o tools/exp/$name.so paper_2104_09404_b200/csrc/mgrit_phi.cu 2>&1 | grep -E "error" 
echo "$name done"
