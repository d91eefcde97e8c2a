# ncu --set full of the scan kernel (pip_tile_kernel) on c4 (1e8 points); c4 launch list
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/prof; rm -rf $O; mkdir -p $O
timeout 300 python tools/prof_kernel.py --workload c4 --points 100000000 --reps 2 > $O/plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pip_tile -s 1 -c 1 -o $O/full_c4 python tools/prof_kernel.py --workload c4 --points 100000000 --reps 2 > $O/ncu_c4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv python tools/prof_kernel.py --workload c4 --points 100000000 --reps 2 > $O/ncu_l4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1.csv python tools/prof_kernel.py --workload c1 --points 1000000 --reps 2 > $O/ncu_l1.log 2>&1
ls -la $O
