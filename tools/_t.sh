# scratch driver for gpurun calls (the last command run on the GPU box)
for w in "0 3000" "280000 3000"; do for n in 16 15 16 15; do echo -n "ndw=$n "; SOM_TIER_NDW=$n python tools/lib_ab.py $w; done; done > gpurun_out/ab_ndw15.log 2>&1
