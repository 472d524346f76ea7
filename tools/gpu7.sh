timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 6000 -c 400 --csv --log-file gpurun_out/launches_sampled.csv python tools/sampled_run.py cfg3 2100 > gpurun_out/launches_sampled.log 2>&1
tail -2 gpurun_out/launches_sampled.log
