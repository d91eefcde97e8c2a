#!/bin/bash
# ncu --set full capture of the scan kernel (pip_tile) on a single-polygon workload: args tag prof_kernel-args
cd ${GRAFT_REPO_ROOT:-.}
T=$1; shift
O=gpurun_out/ncu_scan_$T; rm -rf $O; mkdir -p $O
timeout 300 python tools/prof_kernel.py "$@" --reps 3 > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pip_tile -s 1 -c 1 -o $O/full python tools/prof_kernel.py "$@" --reps 3 > $O/ncu.log 2>&1
echo rc=$?
