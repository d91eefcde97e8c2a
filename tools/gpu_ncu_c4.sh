#!/bin/bash
# ncu --set full captures on configs[3] (C1): the scan kernel and the radix scatter pass
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/ncu_c4${1:-}; rm -rf $O; mkdir -p $O
A="--workload c4 --points 100000000 --mode 0 --reps 2"
timeout 300 python tools/prof_kernel.py $A > $O/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pip_tile -s 1 -c 1 -o $O/scan python tools/prof_kernel.py $A > $O/ncu_scan.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rk_scatter -s 2 -c 2 -o $O/scatter python tools/prof_kernel.py $A > $O/ncu_scatter.log 2>&1
echo "rc=$?"
