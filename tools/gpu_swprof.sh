cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/prof_kernel.py --workload c2 --n 1000000 --points 1000000 --reps 2 > gpurun_out/plain_c2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pip_tile -s 1 -c 1 -o gpurun_out/prof_sw python tools/prof_kernel.py --workload c2 --n 1000000 --points 1000000 --reps 2 > gpurun_out/ncu_sw.log 2>&1
echo done
