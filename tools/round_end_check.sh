set -x
timeout 1800 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
# compute-sanitizer is closed on the GPU pool since round 2 (runs under it left GPUs needing a reset);
# tools/run_sanitizer.sh + tools/sanitize_cases.py remain for pools where it is allowed
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --clock-control none -k regex:som_train --csv --log-file gpurun_out/traffic_c3.csv python tools/c3_window.py 0 500000 > gpurun_out/traffic_c3.log 2>&1
python tools/traffic_json.py gpurun_out/traffic_c3.csv gpurun_out/traffic_c3.json > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-baseline > gpurun_out/bench_ncu.log 2>&1
BENCH_ONE_DEVICE=1 BENCH_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c2 --epochs 1 --steps 1 --warmup 3 --c5-docs 400000 --c4-steps 100 --no-baseline --table3-steps 0 --batch-epochs 0 --c2-steps 0 > gpurun_out/bench_n2.log 2>&1; echo rc=$? >> gpurun_out/bench_n2.log
