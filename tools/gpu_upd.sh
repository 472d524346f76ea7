timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/update_profile.py 2>&1 | grep -E "cfg3|^\[" 
timeout 600 python bench.py --no-m-sweep --no-find-microbench --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-240; grep -o '"phase_ms_per_step": {[^}]*}' gpurun_out/bench.log; grep -o '"e2e": {[^}]*}' gpurun_out/bench.log
