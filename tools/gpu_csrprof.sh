cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/prof_kernel.py --workload c3 --polys 1000000 --reps 2 > gpurun_out/plain_c3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pip_csr_tile -s 1 -c 1 -o gpurun_out/prof_c3b python tools/prof_kernel.py --workload c3 --polys 1000000 --reps 2 > gpurun_out/ncu_c3.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/prof_kernel.py --workload c3 --polys 1000000 --reps 2 > gpurun_out/ncu_c3l.log 2>&1
echo done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python tools/prof_kernel.py --workload c5 --polys 100000 --reps 2 > gpurun_out/ncu_c5l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pip_csr_tile -s 1 -c 1 -o gpurun_out/prof_c5b python tools/prof_kernel.py --workload c5 --polys 100000 --reps 2 > gpurun_out/ncu_c5.log 2>&1
