#!/bin/bash
# GPU tests, then the e2e keys of the default sweep and config 4.
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/e2e; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.log
for w in c2_sweep c4; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err
  python -c "import json; d=json.load(open('$O/bench_$w.json')); print('$w', '%.3g'%d['value'], d['ms_per_step'], 'e2e %.3g'%d['e2e']['value'], d['e2e']['ms_per_step'])"
done
