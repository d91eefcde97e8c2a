#!/bin/bash
# Evidence part 2: GPU tests, smoke, bench lines for every config / mode, the
# reference arm, launch lists (each command first exits 0 without ncu).
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/evidence; mkdir -p $O
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 1800 python -m pytest tests -m gpu -q --timeout 1200 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
fi
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
for w in c1 c3 c5; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 900 python bench.py --workload c2_sweep --steps 3 --warmup 3 > $O/bench_c2_sweep.json 2> $O/bench_c2_sweep.err
for m in 1 2; do timeout 900 python bench.py --mode $m --steps 5 --warmup 3 --no-sweep > $O/bench_c4_mode$m.json 2> $O/bench_c4_mode$m.err; done
for w in c3 c5; do for m in 1 2; do timeout 900 python bench.py --workload $w --mode $m --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_${w}_mode$m.json 2> $O/bench_${w}_mode$m.err; done; done
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep > $O/plain_bench.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep > $O/ncu_launch.log 2>&1
timeout 600 python bench.py --workload c1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain_c1.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1.csv python bench.py --workload c1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch_c1.log 2>&1
timeout 600 python bench.py --workload c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain_c3.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --workload c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch_c3.log 2>&1
echo done
