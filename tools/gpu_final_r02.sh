# round-2 evidence: full bench line, per-batch update profile, ncu launch list and full captures
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_full.log | cut -c1-200
timeout 300 python tools/update_profile.py > gpurun_out/update_profile.log 2>&1; echo "uprof rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 1500 --csv --log-file gpurun_out/launches_cfg3.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-find-microbench --no-m-sweep --no-ref-full --no-cfg4 --no-sharded-anchor > gpurun_out/launches_bench.log 2>&1; echo "ncu list rc=$?"
ncu --set full --cache-control none --clock-control none --import-source on -k k_update_batch -s 1500 -c 2 -o gpurun_out/prof_update_warm_r02f -f python tools/profile_run.py cfg3 1600 > gpurun_out/ncu_u.log 2>&1; echo "ncu upd rc=$?"
ncu --set full --clock-control none --import-source on -k k_update_batch -s 1500 -c 2 -o gpurun_out/prof_update_r02f -f python tools/profile_run.py cfg3 1600 > gpurun_out/ncu_u2.log 2>&1; echo "ncu upd cold rc=$?"
ncu --set full --clock-control none --import-source on -k regex:find_small -s 1500 -c 2 -o gpurun_out/prof_find_small_r02f -f python tools/sampled_run.py cfg3 1600 > gpurun_out/ncu_f.log 2>&1; echo "ncu find rc=$?"
