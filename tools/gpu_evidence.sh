# Round evidence: tests, bench lines for every config, launch list of the bench
# command, one full ncu capture of the dominant kernel per workload family.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ev
O=gpurun_out/ev
nvidia-smi > $O/nvidia-smi.txt 2>&1; lscpu > $O/lscpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in c1 c4 c3 c5; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
# launch list of the bench command (serialised, cold-cache: compare shares)
timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/plain_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
# full capture: dominant kernel of the default workload (n = 1e6 star, 1e6 points), c4 and c3
timeout 300 python tools/prof_kernel.py --workload c2 --n 1000000 --points 1000000 --reps 2 > $O/plain_c2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pip_tile -s 1 -c 1 -o $O/full_sweep_n1e6 python tools/prof_kernel.py --workload c2 --n 1000000 --points 1000000 --reps 2 > $O/ncu_full_sweep.log 2>&1
timeout 300 python tools/prof_kernel.py --workload c3 --polys 1000000 --reps 2 > $O/plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pip_csr -s 1 -c 1 -o $O/full_c3 python tools/prof_kernel.py --workload c3 --polys 1000000 --reps 2 > $O/ncu_full_c3.log 2>&1
echo done
