#!/bin/bash
# Key ncu counters of the C3 sweep kernel for each development variant:
#   scripts/var_ncu.sh build/var_a.so build/var_b.so ...  -> gpurun_out/var_ncu/<name>.txt
mkdir -p gpurun_out/var_ncu
for lib in "$@"; do
  name=$(basename $lib .so)
  COINFER_LIB=$PWD/$lib ncu --clock-control none -k regex:solve_small -c 1 \
    --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread \
    python scripts/quick_sweep.py 300000 > gpurun_out/var_ncu/$name.txt 2>&1
  echo "== $name"; grep -E "duration|inst_executed|fp64|issue_active|stalled|warps_active|registers" gpurun_out/var_ncu/$name.txt | awk '{print $1, $(NF)}'
done
