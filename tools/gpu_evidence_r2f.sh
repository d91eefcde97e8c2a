#!/bin/bash
# Round-2 (session f) evidence on one B200 (run under gpurun): GPU tests, bench lines, launch
# lists, ncu --set full captures of the dominant kernel per config.
# Summarise afterwards with: python tools/summarize_profiles.py gpurun_out/evidence <round tag>
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/evidence
rm -rf $O; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1; lscpu > $O/lscpu.txt 2>&1
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
fi
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in c1 c3 c5; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 900 python bench.py --workload c2_sweep --steps 3 --warmup 3 > $O/bench_c2_sweep.json 2> $O/bench_c2_sweep.err
for m in 1 2; do timeout 900 python bench.py --mode $m --steps 5 --warmup 3 --no-sweep > $O/bench_c4_mode$m.json 2> $O/bench_c4_mode$m.err; done
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
# the driver's torchrun launch at N=1 (NCCL process group, rank-0 line) and smoke()
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 > $O/bench_torchrun1.json 2> $O/bench_torchrun1.err; echo "torchrun rc=$?" >> $O/bench_torchrun1.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
# launch lists (each command first exits 0 without ncu)
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep > $O/plain_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep > $O/ncu_launch.log 2>&1
timeout 600 python bench.py --workload c1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain_c1.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1.csv python bench.py --workload c1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch_c1.log 2>&1
timeout 600 python bench.py --workload c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain_c3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --workload c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch_c3.log 2>&1
# full captures of the dominant kernels (names <workload>_<mode> are the keys bench.py reads)
cap() { # name, kernel regex, prof_kernel args
  timeout 300 python tools/prof_kernel.py $3 --reps 2 > $O/plain_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o $O/full_$1 python tools/prof_kernel.py $3 --reps 2 > $O/ncu_full_$1.log 2>&1
}
cap c4_C1 pip_tile "--workload c4 --points 100000000 --mode 0"
cap c4_C2 pip_tile "--workload c4 --points 100000000 --mode 1"
cap c4_Robust pip_tile "--workload c4 --points 100000000 --mode 2"
cap c1_C1 pip_tile "--workload c1 --points 1000000 --mode 0"
cap c2_sweep_C1 pip_tile "--workload c2 --n 1000000 --points 1000000 --mode 0"
cap c3_C1 pip_csr_tile "--workload c3 --polys 1000000 --mode 0"
cap c5_C1 pip_csr_tile "--workload c5 --polys 100000 --mode 0"
echo done
