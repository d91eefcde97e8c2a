#!/bin/bash
# One ncu --set full capture of the CSR kernel on config 3 (args: tag kernel-regex [workload polys mode])
cd ${GRAFT_REPO_ROOT:-.}
T=${1:-fast}; K=${2:-pip_csr_fast}; W=${3:-c3}; P=${4:-1000000}; M=${5:-0}
O=gpurun_out/ncu_$T; rm -rf $O; mkdir -p $O
timeout 300 python tools/prof_kernel.py --workload $W --polys $P --mode $M --reps 2 > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 -o $O/full python tools/prof_kernel.py --workload $W --polys $P --mode $M --reps 2 > $O/ncu.log 2>&1
echo "rc=$?"; tail -2 $O/ncu.log
