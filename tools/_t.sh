# scratch driver for gpurun calls (the last command run on the GPU box)
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
