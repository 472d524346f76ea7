# A/B the variant libraries (run under gpurun): quick cfg3 bench per variant
for so in paper_1503_08294_b200/variants/*.so; do
  n=$(basename $so .so)
  GS_LIB_PATH=$so timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-find-microbench --no-m-sweep --no-cfg4 --no-sharded-anchor --steps 5 --warmup 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', round(d['ms_per_step'],1), 'find', round(d['phase_ms_per_step']['find'],1), 'upd', round(d['phase_ms_per_step']['update'],1))"
done
