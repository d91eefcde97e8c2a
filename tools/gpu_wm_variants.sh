#!/bin/bash
# A/B of library variants (lib/<variant>) per workload and mode: step and scan-kernel ms
cd ${GRAFT_REPO_ROOT:-.}
for v in ${VARIANTS:-""}; do [ "$v" = default ] && v=""; for w in ${WORKLOADS:-c4 c1}; do for m in ${MODES:-0 1}; do
POLYCAST_LIB_VARIANT=$v timeout 300 python bench.py --workload $w --mode $m --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/wm.json 2> gpurun_out/wm.err || tail -3 gpurun_out/wm.err
python -c "import json; d=json.load(open('gpurun_out/wm.json')); print('variant=$v $w mode $m', 'ms/step', round(d['ms_per_step'],4), 'kernel ms', round(d['roofline']['kernel_ms_per_step'],4))"
done; done; done
