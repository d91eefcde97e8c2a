#!/bin/bash
# One ncu --set full capture of the CSR tile kernel on config 3 (and config 5).
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/ncuc3; mkdir -p $O
timeout 300 python tools/prof_kernel.py --workload c3 --polys 1000000 --reps 2 > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pip_csr_tile -s 1 -c 1 -o $O/full_c3 python tools/prof_kernel.py --workload c3 --polys 1000000 --reps 2 > $O/ncu.log 2>&1
echo "rc=$?"; tail -3 $O/ncu.log
