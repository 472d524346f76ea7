nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash tools/gpu_round.sh
timeout 600 python tools/update_profile.py > gpurun_out/update_profile.log 2>&1; echo "uprof rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 1500 --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-find-microbench --no-m-sweep --no-ref-full --no-cfg4 --no-sharded-anchor > gpurun_out/launches_bench.log 2>&1; echo "ncu rc=$?"
