timeout 900 python -m pytest tests/test_gpu_tier.py tests/test_gpu_sampling.py tests/test_gpu_trajectory_pins.py -q -x > gpurun_out/t_tier.log 2>&1; echo rc=$? >> gpurun_out/t_tier.log
for i in 1 2; do python tools/c3_window.py 0 500000; done > gpurun_out/c3_full.log 2>&1
