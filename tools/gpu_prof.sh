# ncu evidence for the bench workload (run under gpurun; 1 GPU)
set -x
timeout 300 python tools/profile_run.py cfg3 > gpurun_out/profile_run.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 10000 -c 3000 --csv \
  --log-file gpurun_out/launches_cfg3.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
  > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update_batch -s 3000 -c 2 \
  -o gpurun_out/prof_update python tools/profile_run.py cfg3 2000 > gpurun_out/ncu_update.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:find_ -s 3000 -c 2 \
  -o gpurun_out/prof_find python tools/profile_run.py cfg3 2000 > gpurun_out/ncu_find.log 2>&1
ls -la gpurun_out
