timeout 900 python -m pytest tests/test_gpu_tier.py -q -x -k "exchange_variants or late_window" > gpurun_out/t_x.log 2>&1; echo rc=$? >> gpurun_out/t_x.log
