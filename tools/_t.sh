# scratch driver for gpurun calls (the last command run on the GPU box)
for L in A V A V; do SOM_LIB=ab/libsom_$L.so python tools/sweep_grid.py c2 20 128; done > gpurun_out/ab_c2d.log 2>&1
