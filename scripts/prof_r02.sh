#!/bin/bash
# Round-2 profiling pass on the GPU box (gpurun).  Writes text summaries under
# gpurun_out/ (the .ncu-rep files stay on the box: they exceed gpurun's limit):
#   <tag>_full.txt / _lines.csv   ncu --set full (+source) of the 1M-instance C3 solve
#   <tag>_phase.txt               per-phase SM cycles (build/libphase.so, -DCFB_PHASE_TIMING)
#   <tag>_c4.txt / <tag>_c5.txt   ncu --set full of the C4 large-path kernels / one C5 launch
TAG=${1:-r02}
R=/tmp/ncu_$TAG; mkdir -p $R
set -x
ncu --set full --import-source on --clock-control none -k regex:solve_small -c 1 \
    -o $R/full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
    > gpurun_out/${TAG}_full.log 2>&1
bash scripts/ncu_summary.sh $R/full.ncu-rep > gpurun_out/${TAG}_full.txt 2>&1
python scripts/ncu_linedump.py $R/full.ncu-rep > gpurun_out/${TAG}_lines.csv 2>&1
[ -f build/libphase.so ] && COINFER_LIB=build/libphase.so python scripts/phase_time.py 100000 50 > gpurun_out/${TAG}_phase.txt 2>&1
if [ -n "$C4" ]; then
  ncu --set full --import-source on --clock-control none -k regex:large -o $R/c4 \
      python scripts/prof_c4.py 4096 > gpurun_out/${TAG}_c4.log 2>&1
  ncu -i $R/c4.ncu-rep --page raw --csv > $R/c4_raw.csv 2>/dev/null
  python scripts/ncu_kernels.py $R/c4_raw.csv > gpurun_out/${TAG}_c4.txt 2>&1
  python scripts/ncu_linedump.py $R/c4.ncu-rep > gpurun_out/${TAG}_c4_lines.csv 2>&1
  ncu --set full --import-source on --clock-control none -k regex:online --launch-skip 1 -c 1 -o $R/c5 \
      python scripts/bench_online.py 4096 3000 light > gpurun_out/${TAG}_c5.log 2>&1
  bash scripts/ncu_summary.sh $R/c5.ncu-rep > gpurun_out/${TAG}_c5.txt 2>&1
  python scripts/ncu_linedump.py $R/c5.ncu-rep > gpurun_out/${TAG}_c5_lines.csv 2>&1
fi
true
