# scratch driver for gpurun calls (the last command run on the GPU box)
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:som_train --csv --log-file gpurun_out/traffic_c3.csv python tools/c3_window.py 0 500000 > gpurun_out/traffic_c3.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-baseline > gpurun_out/bench_ncu.log 2>&1
