cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out/g1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/g1/bench_c4.json 2> gpurun_out/g1/bench_c4.err; echo "bench rc=$?"
bash tools/gpu_c3only.sh > gpurun_out/g1/c3.txt 2>&1
bash tools/gpu_ncu_c3.sh > gpurun_out/g1/ncu_c3.txt 2>&1
cp -r gpurun_out/ncuc3 gpurun_out/g1/ 2>/dev/null
