timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-find-microbench --no-m-sweep --no-cfg4 --no-sharded-anchor --no-ref-full --steps 5 --warmup 2 > gpurun_out/b$i.log 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/b$i.log; done
echo base; timeout 300 python tools/cfg_timing.py cfg1 cfg2
for v in c8 c4; do echo $v; GS_LIB_PATH=paper_1503_08294_b200/variants/$v.so timeout 300 python tools/cfg_timing.py cfg1 cfg2 cfg3; done
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report all --error-exitcode 9 python tools/race_update.py 300 > gpurun_out/racecheck_update.log 2>&1; echo "racecheck update rc=$?"; tail -2 gpurun_out/racecheck_update.log
