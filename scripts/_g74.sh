for v in q1 q2 q3; do echo $v >> gpurun_out/g74.txt; COINFER_LIB=build/var_$v.so timeout 300 python scripts/m100_time.py 100000 100 >> gpurun_out/g74.txt 2>&1; done
