timeout 1500 python scripts/var_bench.py build/var_p3.so > gpurun_out/g73.txt 2>&1
for v in p3 p3off; do echo $v >> gpurun_out/g73.txt; for M in 100 90 84; do COINFER_LIB=build/var_$v.so timeout 300 python scripts/m100_time.py 100000 $M >> gpurun_out/g73.txt 2>&1; done; done
