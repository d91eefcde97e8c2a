cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/q1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q1/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/q1/bench_c4.json 2> gpurun_out/q1/bench_c4.err; echo "bench c4 rc=$?"
timeout 900 python bench.py --workload c3 --steps 5 --warmup 3 > gpurun_out/q1/bench_c3.json 2> gpurun_out/q1/bench_c3.err; echo "bench c3 rc=$?"
timeout 900 python bench.py --workload c1 --steps 5 --warmup 3 > gpurun_out/q1/bench_c1.json 2> gpurun_out/q1/bench_c1.err; echo "bench c1 rc=$?"
