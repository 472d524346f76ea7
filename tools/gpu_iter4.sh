# iteration: GPU tests, a profiling-variant per-batch profile (if built), two short benches
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
for v in paper_1503_08294_b200/variants/*.so; do [ -f "$v" ] && GS_LIB_PATH=$v timeout 300 python tools/update_profile.py > gpurun_out/uprof_v.log 2>&1 && grep -A12 "first tenth" gpurun_out/uprof_v.log; break; done
for i in 1 2; do timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-find-microbench --no-m-sweep --no-cfg4 --no-sharded-anchor --no-ref-full --steps 5 --warmup 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), {k: round(v,1) for k,v in d['phase_ms_per_step'].items()})"; done
tail -2 gpurun_out/pytest_gpu.log
