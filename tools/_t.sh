# scratch driver for gpurun calls (the last command run on the GPU box)
timeout 900 python tools/sweep_tier_plan.py 3000 > gpurun_out/sweep_plan.log 2>&1
