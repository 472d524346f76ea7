set -x
timeout 300 python tools/find_bench.py 1000000 10000 100000 1000000 --mode 1 > gpurun_out/find_bench.log 2>&1; cat gpurun_out/find_bench.log
timeout 300 python tools/find_bench.py 1000000 10000 100000 --mode 0 --reps 2 > gpurun_out/find_bench_exact.log 2>&1; cat gpurun_out/find_bench_exact.log
timeout 600 ncu --set full --clock-control none --import-source on -k k_filter -c 1 -o gpurun_out/prof_filter -f python tools/find_bench.py 1000000 100000 --reps 1 > gpurun_out/ncu_filter.log 2>&1; tail -2 gpurun_out/ncu_filter.log
timeout 600 ncu --set full --clock-control none --import-source on -k k_update_batch -s 1500 -c 1 -o gpurun_out/prof_update -f python tools/profile_run.py cfg3 1600 > gpurun_out/ncu_update.log 2>&1; tail -2 gpurun_out/ncu_update.log
timeout 600 ncu --set full --clock-control none --import-source on -k find_small_kernel -s 1500 -c 1 -o gpurun_out/prof_find_small -f python tools/profile_run.py cfg3 1600 > gpurun_out/ncu_find_small.log 2>&1; tail -2 gpurun_out/ncu_find_small.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 8000 -c 1500 --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-find-microbench > gpurun_out/launches_bench.log 2>&1; tail -2 gpurun_out/launches_bench.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -3 gpurun_out/bench.log
