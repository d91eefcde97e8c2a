#!/bin/bash
# CSR kernel change check: parity (GPU parity suite's CSR tests, band fuzz CSR,
# full-size fast == exact on c3 / c5) and the c3 / c5 bench lines per mode.
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/csr; mkdir -p $O
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_band_fuzz.py -k "csr or config3 or config5 or footprint" > $O/pytest_parity.txt 2>&1; echo "parity rc=$?"; tail -2 $O/pytest_parity.txt
timeout 900 python -m pytest -q -x -m gpu tests/test_full_parity.py -k "fast_vs_exact_csr" > $O/pytest_full.txt 2>&1; echo "full rc=$?"; tail -2 $O/pytest_full.txt
for w in c3 c5; do for m in 0 1 2; do
timeout 600 python bench.py --workload $w --mode $m --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/b_${w}_$m.json 2>/dev/null
python -c "import json; d=json.load(open('$O/b_${w}_$m.json')); r=d['roofline']; print('$w m$m', round(d['ms_per_step'],4), round(r.get('kernel_ms_per_step') or 0,4), r['frac'])"
done; done
