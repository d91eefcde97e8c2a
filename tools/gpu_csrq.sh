cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "prefilter or scatter or fast_path or csr or config3 or config5 or golden or multi_shard or device_pointer or adversarial" > gpurun_out/pytest_gpu_csr.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_csr.log
for w in c3 c5; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
echo done
