# ncu captures of the update kernel: one cascade batch (~100) and one steady batch (1500), warm L2
T=${GS_TAG:-r02b}
ncu --set full --cache-control none --clock-control none --import-source on -k k_update_batch -s 100 -c 1 -o gpurun_out/prof_upd_cascade_$T -f python tools/profile_run.py cfg3 110 > gpurun_out/ncu_upd_c.log 2>&1; echo "c rc=$?"
ncu --set full --cache-control none --clock-control none --import-source on -k k_update_batch -s 1500 -c 1 -o gpurun_out/prof_upd_steady_$T -f python tools/profile_run.py cfg3 1510 > gpurun_out/ncu_upd_s.log 2>&1; echo "s rc=$?"
