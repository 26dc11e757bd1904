# scratch driver for gpurun calls (the last command run on the GPU box)
for w in "0 3000" "280000 3000"; do for L in A B A B; do SOM_LIB=ab/libsom_$L.so python tools/lib_ab.py $w; done; done > gpurun_out/ab_k10g.log 2>&1
