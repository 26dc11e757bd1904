timeout 1200 python -m pytest tests/test_gpu_tier.py tests/test_gpu_train_csr.py tests/test_gpu_sharded.py tests/test_gpu_trajectory_pins.py tests/test_gpu_sampling.py tests/test_gpu_zero_rows.py -q -x > gpurun_out/t_k.log 2>&1; echo rc=$? >> gpurun_out/t_k.log
for i in 1 2; do python tools/c3_window.py 0 500000; done > gpurun_out/c3_full.log 2>&1
