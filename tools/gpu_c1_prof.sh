#!/bin/bash
# configs[0] pipeline: launch list + full captures of the non-scan kernels
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/c1prof; rm -rf $O; mkdir -p $O
A="--workload c1 --points 1000000 --mode 0 --reps 3"
timeout 300 python tools/prof_kernel.py $A > $O/plain.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/prof_kernel.py $A > $O/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prep_small|rk_|finalize" -s 5 -c 5 -o $O/full python tools/prof_kernel.py $A > $O/ncu_full.log 2>&1
echo rc=$?
