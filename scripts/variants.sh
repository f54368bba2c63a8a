#!/bin/bash
# Development variants of the N=4 solver: scripts/variants.sh NAME "-DFLAG=.. ..." [NAME "FLAGS"]...
# Builds build/var_NAME.so (only the N=4 instantiations: fast compiles); the
# objects other than solve_small are compiled once into build/_common.
# Time and check them on the GPU with scripts/var_bench.py build/var_*.so.
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=$ROOT/paper_2206_06304_b200/csrc
F="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -Xcompiler -fPIC -DCFB_ONLY_N=4"
mkdir -p $ROOT/build/_common
for f in capi solve_large online probe baselines generate oracles; do
  o=$ROOT/build/_common/$f.o
  if [ ! -f $o ] || [ $SRC/$f.cu -nt $o ] || [ $SRC/solve_core.cuh -nt $o ] || [ $SRC/device_common.cuh -nt $o ]; then
    nvcc $F -c $SRC/$f.cu -o $o &
  fi
done
wait
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  ( nvcc $F $flags -Xptxas -v -c $SRC/solve_small.cu -o $ROOT/build/_var_$name.o 2> $ROOT/build/var_$name.ptxas.log &
    for sh in 0 1 2; do nvcc $F $flags -c $SRC/solve_pipe$sh.cu -o $ROOT/build/_var_${name}_p$sh.o 2>> $ROOT/build/var_$name.pipe.log & done
    wait
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $ROOT/build/var_$name.so $ROOT/build/_var_$name.o \
      $ROOT/build/_var_${name}_p{0,1,2}.o \
      $ROOT/build/_common/{capi,solve_large,online,probe,baselines,generate,oracles}.o -lcudart &&
    echo "built var_$name" ) &
done
wait
