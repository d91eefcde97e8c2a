#!/bin/bash
# Scan-kernel change check: single-polygon parity (GPU parity suite, band fuzz,
# full-size fast == exact on the single configs) and c4 / c1 / sweep bench lines.
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/scan; mkdir -p $O
timeout 1200 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_band_fuzz.py tests/test_acceptance_gpu.py > $O/pytest_parity.txt 2>&1; echo "parity rc=$?"; tail -2 $O/pytest_parity.txt
timeout 1200 python -m pytest -q -x -m gpu tests/test_full_parity.py -k "fast_vs_exact_single" > $O/pytest_full.txt 2>&1; echo "full rc=$?"; tail -2 $O/pytest_full.txt
for w in ${WORKLOADS:-c4 c1 c2_sweep}; do for m in ${MODES:-0}; do
timeout 600 python bench.py --workload $w --mode $m --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep > $O/b_${w}_$m.json 2>/dev/null
python -c "import json; d=json.load(open('$O/b_${w}_$m.json')); r=d['roofline']; print('$w m$m', round(d['ms_per_step'],4), round(r.get('kernel_ms_per_step') or 0,4), '%.3e'%d['value'])"
done; done
