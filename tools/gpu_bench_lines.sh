#!/bin/bash
# Bench lines only (after tools/summarize_profiles.py refreshed profiles/ncu_kernels.json)
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/benchlines; rm -rf $O; mkdir -p $O
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in c1 c3 c5; do timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err; done
for m in 1 2; do for w in c3 c5; do timeout 900 python bench.py --workload $w --mode $m --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_${w}_mode$m.json 2> $O/bench_${w}_mode$m.err; done; done
timeout 900 python bench.py --workload c2_sweep --steps 3 --warmup 3 > $O/bench_c2_sweep.json 2> $O/bench_c2_sweep.err
for m in 1 2; do timeout 900 python bench.py --mode $m --steps 5 --warmup 3 --no-sweep > $O/bench_c4_mode$m.json 2> $O/bench_c4_mode$m.err; done
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 > $O/bench_torchrun1.json 2> $O/bench_torchrun1.err
echo done
