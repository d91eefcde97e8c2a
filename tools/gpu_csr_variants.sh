#!/bin/bash
# A/B of CSR tile-kernel build variants (lib/<variant>): c3 / c5 kernel time per mode
cd ${GRAFT_REPO_ROOT:-.}
for v in ${VARIANTS:-"" w64m8 w64m7 w96m6}; do [ "$v" = default ] && v=""; for w in ${WORKLOADS:-c3 c5}; do for m in ${MODES:-0}; do
POLYCAST_LIB_VARIANT=$v timeout 300 python bench.py --workload $w --mode $m --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('variant=$v $w m$m', 'ms/step', round(d['ms_per_step'],4), 'kernel ms', round(d['roofline']['kernel_ms_per_step'],4))"
done; done; done
