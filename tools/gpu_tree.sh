#!/bin/bash
# Segment-tree path: parity tests, then the sweep with the tree on / off.
mkdir -p gpurun_out/tree
timeout 900 python -m pytest tests/test_tree.py -x -q > gpurun_out/tree/tests.log 2>&1
echo "tree tests rc=$?"; tail -25 gpurun_out/tree/tests.log
timeout 600 python tools/prof_kernel.py --workload c2 --n 1000000 --points 1000000 --reps 2 > gpurun_out/tree/prof.log 2>&1; tail -5 gpurun_out/tree/prof.log
timeout 900 python bench.py --steps 3 --no-e2e --no-cpu-baseline 2> gpurun_out/tree/bench.err | cut -c1-300
tail -5 gpurun_out/tree/bench.err
