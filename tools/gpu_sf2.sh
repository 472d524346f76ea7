ncu --set full --clock-control none --import-source on -k regex:find_small -s 1500 -c 2 -o gpurun_out/prof_sf_engine -f python tools/sampled_run.py cfg3 1600 > gpurun_out/ncu_sf.log 2>&1
tail -1 gpurun_out/ncu_sf.log
