# scratch driver for gpurun calls (the last command run on the GPU box)
for i in 1 2; do timeout 900 python -m pytest tests/test_gpu_sharded.py -q -x -k csr_kernels > gpurun_out/t_sh$i.log 2>&1; echo rc=$? >> gpurun_out/t_sh$i.log; done
