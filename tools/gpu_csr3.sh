cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "csr or config3 or config5 or golden or multi_shard or device_pointer" > gpurun_out/pytest_gpu_csr.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_csr.log
for w in c3 c5; do timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
timeout 300 python tools/prof_kernel.py --workload c3 --polys 200000 --reps 2 > gpurun_out/plain_c3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pip_csr_warp -s 1 -c 1 -o gpurun_out/prof_c3b python tools/prof_kernel.py --workload c3 --polys 200000 --reps 2 > gpurun_out/ncu_c3.log 2>&1
echo done
