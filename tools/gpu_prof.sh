# ncu evidence for profiles/ (run under gpurun; 1 GPU)
ncu --set full --clock-control none --import-source on -k k_update_batch -s 1500 -c 2 -o gpurun_out/prof_update -f python tools/profile_run.py cfg3 1600 > gpurun_out/ncu_update.log 2>&1
ncu --set full --cache-control none --clock-control none --import-source on -k k_update_batch -s 1500 -c 2 -o gpurun_out/prof_update_warm -f python tools/profile_run.py cfg3 1600 > gpurun_out/ncu_update_warm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:find_small -s 1500 -c 2 -o gpurun_out/prof_find_small -f python tools/sampled_run.py cfg3 1600 > gpurun_out/ncu_find_small.log 2>&1
ncu --set full --clock-control none --import-source on -k k_cloud_sample -s 20 -c 1 -o gpurun_out/prof_sample -f python tools/sampled_run.py cfg3 1600 > gpurun_out/ncu_sample.log 2>&1
ncu --set full --clock-control none --import-source on -k k_filter -c 1 -o gpurun_out/prof_filter_1e6 -f python tools/find_bench.py 1000000 1000000 --reps 1 > gpurun_out/ncu_filter.log 2>&1
ncu --set full --clock-control none --import-source on -k k_filter -c 1 -o gpurun_out/prof_filter_1e5 -f python tools/find_bench.py 1000000 100000 --reps 1 >> gpurun_out/ncu_filter.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 1500 --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-find-microbench --no-m-sweep > gpurun_out/launches_bench.log 2>&1
ls -la gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_grid_query -c 1 -o gpurun_out/prof_grid_query -f python tools/find_bench.py 1000000 1000000 --mode 4 --reps 1 > gpurun_out/ncu_grid.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_grid.csv python tools/find_bench.py 1000000 10000 1000000 --mode 4 --reps 1 >> gpurun_out/ncu_grid.log 2>&1
