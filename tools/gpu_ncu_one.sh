#!/bin/bash
# One ncu --set full capture of one kernel: gpu_ncu_one.sh <tag> <kernel regex> <prof_kernel.py args...>
cd ${GRAFT_REPO_ROOT:-.}
T=$1; K=$2; shift 2
O=gpurun_out/ncu1; mkdir -p $O
timeout 300 python tools/prof_kernel.py "$@" --reps 2 > $O/$T.plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o $O/$T python tools/prof_kernel.py "$@" --reps 2 > $O/$T.ncu.log 2>&1
echo "$T rc=$?"
