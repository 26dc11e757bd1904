timeout 600 python -m pytest tests/test_gpu_map_tc.py -q -x -s -k many_work > gpurun_out/t_tc2.log 2>&1; echo rc=$? >> gpurun_out/t_tc2.log
