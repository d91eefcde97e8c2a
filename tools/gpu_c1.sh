cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "bucket or config1 or adversarial or golden or config2" > gpurun_out/pytest_c1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c1.log
timeout 600 python bench.py --workload c1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --workload c1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain_c1b.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv python bench.py --workload c1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_c1.log 2>&1
echo done
