cd ${GRAFT_REPO_ROOT:-.}
for b in -1 0; do for w in c1 c2_sweep; do
timeout 600 python bench.py --workload $w --bucket $b --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print('bucket $b $w', '%.4g'%d['value'], 'ms/step', round(d['ms_per_step'],4), 'kernel', round(d['roofline'].get('kernel_ms_per_step') or 0,4), [ (s.get('n'), s.get('kernel_ms')) for s in (d.get('sweep') or {}).get('per_n',[])][:6] if isinstance(d.get('sweep'),dict) else '')"
done; done
