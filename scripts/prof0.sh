set -x
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
ncu --set full --import-source on --clock-control none -k regex:solve_small -c 1 \
    -o gpurun_out/r02/base python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r02/base_bench.log 2>&1
ncu -i gpurun_out/r02/base.ncu-rep --page source --csv --print-source cuda > gpurun_out/r02/base_src.csv 2>&1
ls -la gpurun_out/r02
