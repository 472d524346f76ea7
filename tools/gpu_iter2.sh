# update-kernel iteration: parity tests, per-batch profile, short bench (run under gpurun)
timeout 900 python -m pytest tests -x -q -m gpu ${GS_TESTS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/update_profile.py > gpurun_out/update_profile.log 2>&1; echo "uprof rc=$?"; head -14 gpurun_out/update_profile.log; grep -A12 "first tenth" gpurun_out/update_profile.log
timeout 600 python bench.py --no-m-sweep --no-find-microbench --no-cpu-baseline --no-ref-full --no-cfg4 --no-sharded-anchor > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300; grep -o '"phase_ms_per_step": {[^}]*}' gpurun_out/bench.log; grep -o '"e2e": {[^}]*}' gpurun_out/bench.log
