#!/bin/bash
# Run on the GPU box (gpurun).  Produces, under gpurun_out/:
#   launches.csv   every kernel launch of a short bench run with its device time
#   full.ncu-rep   one --set full capture of the bench's solve kernel (1M instances)
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:solve_small -c 1 \
    -o gpurun_out/full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
    > gpurun_out/full_bench.log 2>&1
