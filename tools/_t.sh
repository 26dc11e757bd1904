# scratch driver for gpurun calls (the last command run on the GPU box)
for w in "320000 3000" "350000 3000" "450000 3000"; do for L in A R A R; do SOM_TRAIN_TIER=0 SOM_LIB=ab/libsom_$L.so python tools/lib_ab.py $w; done; done > gpurun_out/ab_k4c.log 2>&1
timeout 900 python -m pytest tests/test_gpu_train_csr.py tests/test_gpu_tier.py tests/test_gpu_sharded.py tests/test_gpu_trajectory_pins.py tests/test_gpu_zero_rows.py tests/test_gpu_sampling.py -q -x > gpurun_out/t_k4.log 2>&1; echo rc=$? >> gpurun_out/t_k4.log
