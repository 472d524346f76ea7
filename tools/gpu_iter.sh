# Update-kernel iteration loop (run under gpurun): engine parity tests, a
# quick cfg3 bench line, the per-batch update profile
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_sharded.py tests/test_gpu_runstate.py -x -q -m gpu > gpurun_out/iter_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/iter_tests.log
timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-find-microbench --no-m-sweep --no-cfg4 --no-sharded-anchor --steps 3 --warmup 2 > gpurun_out/iter_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/iter_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms_per_step', d['ms_per_step'], 'phase', d['phase_ms_per_step'], 'upd_us_per_batch', d['roofline'].get('us_per_batch'))"
timeout 300 python tools/update_profile.py cfg3 > gpurun_out/iter_profile.txt 2>&1; echo "profile rc=$?"; tail -14 gpurun_out/iter_profile.txt
