#!/bin/bash
# A/B of scan-kernel build variants (lib/<variant>): c4 / c1 / sweep step and kernel ms
cd ${GRAFT_REPO_ROOT:-.}
for v in ${VARIANTS:-""}; do [ "$v" = default ] && v=""; for w in ${WORKLOADS:-c4 c1}; do
POLYCAST_LIB_VARIANT=$v timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/sv.json 2> gpurun_out/sv.err || tail -3 gpurun_out/sv.err
python -c "import json; d=json.load(open('gpurun_out/sv.json')); print('variant=$v $w', 'ms/step', round(d['ms_per_step'],4), 'kernel ms', round(d['roofline']['kernel_ms_per_step'],4))"
done; done
