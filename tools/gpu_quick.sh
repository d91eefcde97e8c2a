cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/q
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -x > gpurun_out/q/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/q/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q/smoke.log 2>&1; echo "smoke rc=$?"
for w in sweep c3 c4; do
 if [ $w = sweep ]; then a=""; else a="--workload $w"; fi
 timeout 900 python bench.py $a --steps 5 --warmup 3 > gpurun_out/q/bench_$w.json 2> gpurun_out/q/bench_$w.err; echo "bench $w rc=$?"; cut -c1-250 gpurun_out/q/bench_$w.json
done
