#!/bin/bash
# per-n scan rates of the configs[1] sweep for library variants
cd ${GRAFT_REPO_ROOT:-.}
for v in ${VARIANTS:-""}; do [ "$v" = default ] && v=""; for m in ${MODES:-0}; do
POLYCAST_LIB_VARIANT=$v timeout 300 python bench.py --workload c2_sweep --mode $m --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/si.json 2> gpurun_out/si.err || tail -3 gpurun_out/si.err
python -c "import json; d=json.load(open('gpurun_out/si.json')); print('variant=$v mode $m', round(d['ms_per_step'],3), {k: '%.3g' % v for k, v in d['per_item_tests_per_s'].items()})"
done; done
