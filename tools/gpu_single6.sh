cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "not csr and not config3 and not config5 and not fast_path and not prefilter and not scatter" > gpurun_out/pytest_gpu_single.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_single.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_sweep.json 2> gpurun_out/bench_sweep.err
timeout 600 python bench.py --workload c1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo done
