# scratch driver for gpurun calls (the last command run on the GPU box)
SOM_TRACE_CLOCK=1 python tools/trace_tier.py 0 2000 1 > gpurun_out/trace_k10b.log 2>&1
