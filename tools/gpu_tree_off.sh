#!/bin/bash
# The default sweep with the segment tree on (auto) and off (the linear scan only).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/treeoff
for t in -1 0; do
  timeout 900 python bench.py --tree $t --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/treeoff/bench_tree$t.json 2> gpurun_out/treeoff/bench_tree$t.err
  python -c "import json; d=json.load(open('gpurun_out/treeoff/bench_tree$t.json')); r=d['roofline']; print('tree $t', '%.3g'%d['value'], d['ms_per_step'], 'frac %.3g'%r['frac'], r.get('note','')[:40])"
done
