set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python tools/find_bench.py 1000000 10000 100000 1000000 --mode 1 > gpurun_out/find_bench.log 2>&1; echo "fb rc=$?"
cat gpurun_out/find_bench.log
timeout 300 python tools/find_bench.py 1000000 10000 100000 --mode 0 --reps 2 > gpurun_out/find_bench_exact.log 2>&1
cat gpurun_out/find_bench_exact.log
timeout 300 python tools/profile_run.py cfg3 > gpurun_out/profile_run.log 2>&1; cat gpurun_out/profile_run.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/probe_launches.csv python tools/profile_run.py cfg3 15 > gpurun_out/probe.log 2>&1
cat gpurun_out/probe.log | tail -5; cut -c1-200 gpurun_out/probe_launches.csv | tail -40
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_filter -s 2 -c 1 -o gpurun_out/prof_filter python tools/find_bench.py 1000000 100000 --reps 1 > gpurun_out/ncu_filter.log 2>&1
tail -3 gpurun_out/ncu_filter.log
