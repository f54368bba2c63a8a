#!/bin/bash
# Per-instruction execution counts (SourceCounters) of the C3 sweep kernel per variant:
#   scripts/var_src.sh build/var_a.so ...  -> gpurun_out/var_src/<name>.ncu-rep
mkdir -p gpurun_out/var_src
for lib in "$@"; do
  name=$(basename $lib .so)
  COINFER_LIB=$PWD/$lib ncu --clock-control none -k regex:solve_small -c 1 --section SourceCounters --section WarpStateStats \
    --import-source on -o gpurun_out/var_src/$name python scripts/quick_sweep.py 300000 > gpurun_out/var_src/$name.log 2>&1
done
ls -la gpurun_out/var_src
