timeout 600 python -m pytest tests/test_gpu_filter.py tests/test_gpu_find.py -x -q > gpurun_out/pytest_filter.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_filter.log
timeout 300 python tools/find_bench.py 1000000 10000 100000 1000000 --mode 1 > gpurun_out/find_bench.log 2>&1; cut -c1-220 gpurun_out/find_bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k k_filter -c 1 -o gpurun_out/prof_filter -f python tools/find_bench.py 1000000 100000 --reps 1 > gpurun_out/ncu_filter.log 2>&1; tail -1 gpurun_out/ncu_filter.log
