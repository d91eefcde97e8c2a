#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): GPU tests, every bench line,
# launch lists, one ncu --set full capture per hot kernel, the CSV I/O bench.
# Summarise afterwards with: python tools/summarize_profiles.py gpurun_out/evidence <round tag>
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/evidence
rm -rf $O; mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1; lscpu > $O/lscpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in c1 c4 c3 c5; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err; done
for m in 1 2; do timeout 900 python bench.py --mode $m --steps 3 --warmup 3 > $O/bench_sweep_mode$m.json 2> $O/bench_sweep_mode$m.err; done
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python tools/bench_csv.py --rows 10000000 > $O/bench_csv.jsonl 2> $O/bench_csv.err
# launch lists (each command first exits 0 without ncu)
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/plain_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 600 python bench.py --workload c1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/plain_c1.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1.csv python bench.py --workload c1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch_c1.log 2>&1
timeout 600 python bench.py --workload c3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/plain_c3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --workload c3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch_c3.log 2>&1
# segment-tree path: launch list at n = 1e6 and the scan/tree crossover table
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_tree_n1e6.csv python tools/prof_kernel.py --workload c2 --n 1000000 --points 1000000 --reps 1 > $O/ncu_launch_tree.log 2>&1
timeout 600 bash tools/gpu_tree_thr.sh > $O/tree_crossover.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:query_kernel -c 1 -o $O/full_tree_query python tools/prof_kernel.py --workload c2 --n 1000000 --points 1000000 --reps 1 > $O/ncu_full_tree.log 2>&1
# full captures of the hot kernels
# the scan kernel (tree off) on the same inputs, for comparison
timeout 300 python tools/prof_kernel.py --workload c2 --n 1000000 --points 1000000 --reps 2 --tree 0 > $O/plain_c2k.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pip_tile -s 1 -c 1 -o $O/full_sweep_n1e6 python tools/prof_kernel.py --workload c2 --n 1000000 --points 1000000 --reps 2 --tree 0 > $O/ncu_full_sweep.log 2>&1
timeout 300 python tools/prof_kernel.py --workload c4 --points 10000000 --reps 2 --tree 0 > $O/plain_c4k.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pip_tile -s 1 -c 1 -o $O/full_c4 python tools/prof_kernel.py --workload c4 --points 10000000 --reps 2 --tree 0 > $O/ncu_full_c4.log 2>&1
timeout 300 python tools/prof_kernel.py --workload c3 --polys 1000000 --reps 2 > $O/plain_c3k.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pip_csr_tile -s 1 -c 1 -o $O/full_c3 python tools/prof_kernel.py --workload c3 --polys 1000000 --reps 2 > $O/ncu_full_c3.log 2>&1
timeout 300 python tools/prof_kernel.py --workload c5 --polys 100000 --reps 2 > $O/plain_c5k.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pip_csr_tile -s 1 -c 1 -o $O/full_c5 python tools/prof_kernel.py --workload c5 --polys 100000 --reps 2 > $O/ncu_full_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:csv_parse_kernel -c 1 -o $O/full_csv_parse python tools/bench_csv.py --rows 10000000 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full_csv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:emit_format_kernel -c 1 -o $O/full_csv_emit python tools/bench_csv.py --rows 10000000 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_full_emit.log 2>&1
echo done
