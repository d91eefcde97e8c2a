#!/bin/bash
# CSR kernels on one B200: GPU tests, then c3 / c5 bench lines in every mode.
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/csr; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
for w in c3 c5; do for m in 0 1 2; do
  timeout 600 python bench.py --workload $w --mode $m --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_${w}_m$m.json 2> $O/bench_${w}_m$m.err
  python -c "import json,sys; d=json.load(open('$O/bench_${w}_m$m.json')); r=d['roofline']; print('$w m$m', d['ms_per_step'], r.get('kernel_ms_per_step'), r['frac'])"
done; done
