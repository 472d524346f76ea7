# compute-sanitizer memcheck over short runs of every kernel family (1 GPU)
set -x
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_engine.py -x -q -m gpu -k "cfg1 or stress or boundary or winner or errors or floor or remove" > gpurun_out/memcheck_engine.log 2>&1; echo "engine rc=$?"
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_filter.py tests/test_gpu_find.py tests/test_sampler.py -x -q -m gpu > gpurun_out/memcheck_find.log 2>&1; echo "find rc=$?"
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_small_find.py tests/test_gpu_grid_find.py -x -q -m gpu -k "not 100_003 and not 20000" > gpurun_out/memcheck_small_grid.log 2>&1; echo "small+grid rc=$?"
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_engine.py -x -q -m gpu -k "cfg1 or stress" > gpurun_out/racecheck_engine.log 2>&1; echo "racecheck engine rc=$?"
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_small_find.py -x -q -m gpu -k "c_oracle or ties" > gpurun_out/racecheck_small.log 2>&1; echo "racecheck small rc=$?"
timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_find.py -x -q -m gpu -k "golden or oracle" > gpurun_out/racecheck_find.log 2>&1; echo "racecheck find rc=$?"
for f in gpurun_out/memcheck_engine.log gpurun_out/memcheck_find.log gpurun_out/memcheck_small_grid.log gpurun_out/racecheck_find.log gpurun_out/racecheck_engine.log gpurun_out/racecheck_small.log; do echo "== $f"; tail -n 4 $f; done
