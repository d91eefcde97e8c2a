#!/bin/bash
mkdir -p gpurun_out/tree
timeout 600 python tools/prof_kernel.py --workload c2 --n 1000000 --points 1000000 --reps 1 > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tree/launches_n1e6.csv python tools/prof_kernel.py --workload c2 --n 1000000 --points 1000000 --reps 1 > gpurun_out/tree/ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tree/launches_n1e5.csv python tools/prof_kernel.py --workload c2 --n 100000 --points 1000000 --reps 1 > gpurun_out/tree/ncu2.log 2>&1
echo done
