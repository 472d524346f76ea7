# small-n screened find: parity + timing (one B200)
timeout 900 python -m pytest tests/test_gpu_small_find.py -x -q > gpurun_out/sf_tests.log 2>&1; echo "sf tests rc=$?"; tail -3 gpurun_out/sf_tests.log
for mode in 0 3; do timeout 120 python tools/find_bench.py 4096 1000 2000 4000 --mode $mode --reps 20 | cut -c1-120; done
for fs in 1 2 4; do GS_SF_FS=$fs timeout 120 python tools/find_bench.py 4096 2000 --mode 3 --reps 20 | cut -c1-120; done
timeout 300 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-m-sweep --no-find-microbench --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300; grep -o '"phase_ms_per_step": {[^}]*}' gpurun_out/bench.log
