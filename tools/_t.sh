# scratch driver for gpurun calls (the last command run on the GPU box)
python tools/prof_c4.py 200 1 > gpurun_out/c4.log 2>&1
python tools/prof_c4.py 200 0 >> gpurun_out/c4.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:som_train -c 1 -o gpurun_out/k4_c4 python tools/prof_c4.py 100 1 > gpurun_out/ncu_c4.log 2>&1
