# A/B of library variants (lib/<v>) on the bench workloads
cd ${GRAFT_REPO_ROOT:-.}
for v in ${VARIANTS:-"" s3 s4 s6}; do [ "$v" = default ] && v=""; for w in ${WORKLOADS:-c4 c1}; do POLYCAST_LIB_VARIANT=$v timeout 300 python bench.py --workload $w --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e --no-sweep 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant=$v', d['config']['workload'][:24], 'ms/step', round(d['ms_per_step'],4), 'kernel ms', round(d['roofline']['kernel_ms_per_step'],4))"; done; done
