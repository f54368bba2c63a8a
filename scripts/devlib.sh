#!/bin/bash
# Development library: only the N=4 instantiations of the small solver
# (fast to compile), linked into build/libdev.so; use COINFER_LIB=build/libdev.so.
set -e
cd "$(dirname "$0")/../paper_2206_06304_b200/csrc"
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -Xcompiler -fPIC -DCFB_ONLY_N=4"
for f in ${@:-solve_small}; do nvcc $F -c $f.cu -o /tmp/dev_$f.o; done
mkdir -p ../../build
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../build/libdev.so /tmp/dev_capi.o /tmp/dev_solve_small.o /tmp/dev_solve_large.o /tmp/dev_online.o /tmp/dev_probe.o /tmp/dev_baselines.o /tmp/dev_generate.o /tmp/dev_oracles.o -lcudart
