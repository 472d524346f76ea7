for rep in 1 2; do for fs in 2 4 8; do
GS_SF_FS=$fs timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-find-microbench --no-m-sweep --no-cfg4 --no-sharded-anchor --steps 5 --warmup 2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fs=$fs', round(d['ms_per_step'],1), 'find', round(d['phase_ms_per_step']['find'],1), 'upd', round(d['phase_ms_per_step']['update'],1))"
done; done
