#!/bin/bash
# A/B of library variants (lib/<variant>) on configs[3] per mode: step and scan-kernel ms
cd ${GRAFT_REPO_ROOT:-.}
for v in ${VARIANTS:-""}; do [ "$v" = default ] && v=""; for m in ${MODES:-1 2}; do
POLYCAST_LIB_VARIANT=$v timeout 300 python bench.py --mode $m --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > gpurun_out/mv.json 2> gpurun_out/mv.err || tail -3 gpurun_out/mv.err
python -c "import json; d=json.load(open('gpurun_out/mv.json')); print('variant=$v mode $m', 'ms/step', round(d['ms_per_step'],4), 'kernel ms', round(d['roofline']['kernel_ms_per_step'],4))"
done; done
