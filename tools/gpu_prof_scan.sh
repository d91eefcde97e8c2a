# ncu --set full of the scan kernel (pip_tile_kernel) on c4 (1e7 points) and the sweep's n=1e6 star; c4 launch list
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/prof; rm -rf $O; mkdir -p $O
timeout 300 python tools/prof_kernel.py --workload c4 --points 10000000 --reps 2 > $O/plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pip_tile -s 1 -c 1 -o $O/full_c4 python tools/prof_kernel.py --workload c4 --points 10000000 --reps 2 > $O/ncu_c4.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:pip_tile -s 1 -c 1 -o $O/full_n1e6 python tools/prof_kernel.py --workload c2 --n 1000000 --points 1000000 --reps 2 > $O/ncu_n1e6.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv python tools/prof_kernel.py --workload c4 --points 100000000 --reps 2 > $O/ncu_l4.log 2>&1
ls -la $O
