# scratch driver for gpurun calls (the last command run on the GPU box)
SOM_TIER_HANDOVER=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:som_train_tier -c 1 -o gpurun_out/k10_early_v2 python tools/c3_window.py 0 1000 > gpurun_out/ncu_k10.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:som_train_reg -c 1 -o gpurun_out/k2_c2 python tools/trace_train.py c2 128 20000 0 > gpurun_out/ncu_k2.log 2>&1
