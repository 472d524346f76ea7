# round-2 ncu captures of the config-3 hot kernels (run under gpurun; 1 GPU)
T=${GS_TAG:-r02}
ncu --set full --clock-control none --import-source on -k k_update_batch -s 1500 -c 2 -o gpurun_out/prof_update_$T -f python tools/profile_run.py cfg3 1600 > gpurun_out/ncu_update_$T.log 2>&1; echo "upd rc=$?"
ncu --set full --cache-control none --clock-control none --import-source on -k k_update_batch -s 1500 -c 2 -o gpurun_out/prof_update_warm_$T -f python tools/profile_run.py cfg3 1600 > gpurun_out/ncu_update_warm_$T.log 2>&1; echo "updw rc=$?"
ncu --set full --clock-control none --import-source on -k regex:find_small -s 1500 -c 2 -o gpurun_out/prof_find_small_$T -f python tools/sampled_run.py cfg3 1600 > gpurun_out/ncu_find_small_$T.log 2>&1; echo "find rc=$?"
