#!/bin/bash
# Development library: only the N=4 instantiations of the small solver
# (fast to compile), linked into build/libdev.so (or $OUT); use COINFER_LIB=build/libdev.so.
# Extra nvcc flags via $EXTRA (e.g. EXTRA=-DCFB_PHASE_TIMING).
set -e
cd "$(dirname "$0")/../paper_2206_06304_b200/csrc"
OUT=${OUT:-../../build/libdev.so}
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -Xcompiler -fPIC -DCFB_ONLY_N=4 $EXTRA"
T=/tmp/devobj_$$
mkdir -p $T ../../build
pids=()
for f in capi solve_small solve_pipe0 solve_pipe1 solve_pipe2 solve_large online probe baselines generate oracles; do
  nvcc $F -c $f.cu -o $T/$f.o & pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT $T/*.o -lcudart
rm -rf $T
