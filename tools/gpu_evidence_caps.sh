#!/bin/bash
# Evidence part 1 (run first): ncu --set full captures of the dominant kernel per
# config, so tools/summarize_profiles.py can refresh profiles/ncu_kernels.json
# (bench.py's roofline reads it) before the bench lines are taken.
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/evidence; rm -rf $O; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1; lscpu > $O/lscpu.txt 2>&1
cap() { # name, kernel regex, prof_kernel args
  timeout 300 python tools/prof_kernel.py $3 --reps 2 > $O/plain_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o $O/full_$1 python tools/prof_kernel.py $3 --reps 2 > $O/ncu_full_$1.log 2>&1
  echo "cap $1 rc=$?"
}
cap c4_C1 pip_tile "--workload c4 --points 100000000 --mode 0"
cap c4_C2 pip_tile "--workload c4 --points 100000000 --mode 1"
cap c4_Robust pip_tile "--workload c4 --points 100000000 --mode 2"
cap c1_C1 pip_tile "--workload c1 --points 1000000 --mode 0"
cap c2_sweep_C1 pip_tile "--workload c2 --n 1000000 --points 1000000 --mode 0"
cap c3_C1 pip_csr_tile "--workload c3 --polys 1000000 --mode 0"
cap c5_C1 pip_csr_tile "--workload c5 --polys 100000 --mode 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rk_scatter -s 2 -c 2 -o $O/full_sort_c4 python tools/prof_kernel.py --workload c4 --points 100000000 --mode 0 --reps 2 > $O/ncu_full_sort.log 2>&1
echo "sort rc=$?"
