timeout 600 python -m pytest tests/test_gpu_map_tc.py -q -x > gpurun_out/t_tc.log 2>&1; echo rc=$? >> gpurun_out/t_tc.log
for L in N256 N128 N256 N128; do echo "lib $L"; SOM_LIB=ab/libsom_$L.so timeout 300 python tools/prof_map.py 100000 100 20000 2; done > gpurun_out/ab_tc.log 2>&1
for L in N256 N128; do echo "lib $L"; SOM_LIB=ab/libsom_$L.so timeout 300 python tools/prof_map.py 50000 50 10000 2; done >> gpurun_out/ab_tc.log 2>&1
SOM_LIB=ab/libsom_N128.so timeout 600 ncu --set full --clock-control none -k regex:map_tc_kernel -c 1 -o gpurun_out/map_tc128 python tools/prof_map.py 30000 100 20000 1 > gpurun_out/ncu_tc.log 2>&1
