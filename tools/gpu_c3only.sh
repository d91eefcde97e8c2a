cd ${GRAFT_REPO_ROOT:-.}
for m in 0 1 2; do
timeout 600 python bench.py --workload c3 --mode $m --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b.json 2>/dev/null
python -c "import json; d=json.load(open('/tmp/b.json')); r=d['roofline']; print('c3 m$m', d['ms_per_step'], r.get('kernel_ms_per_step'), r['frac'])"
done
