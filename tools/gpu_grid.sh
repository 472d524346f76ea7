timeout 900 python -m pytest tests/test_gpu_grid_find.py tests/test_gpu_engine.py -x -q > gpurun_out/grid_tests.log 2>&1; echo "grid tests rc=$?"; tail -3 gpurun_out/grid_tests.log
for mode in 4; do timeout 300 python tools/find_bench.py 1000000 10000 100000 1000000 --mode $mode --reps 5 | cut -c1-140; done
