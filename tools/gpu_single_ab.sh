#!/bin/bash
# single-polygon path: parity subset + bench c4 / c1 / sweep (quick A/B)
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/single; rm -rf $O; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_full_parity.py -m gpu -q -x --timeout 900 \
  -k "${TESTS:-bucket or config1 or config2 or config4 or scan_chunk or graph or multi_shard or single or golden_vectors or adversarial}" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for w in ${WORKLOADS:-c4 c1}; do
timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sweep > $O/bench_$w.json 2>$O/bench_$w.err
python -c "import json;d=json.loads(open('$O/bench_$w.json').read().strip().splitlines()[-1]);print('$w', '%.4g'%d['value'], 'ms/step', round(d['ms_per_step'],4), 'kernel ms', round(d['roofline'].get('kernel_ms_per_step') or 0,4))"
done
if [ "${LAUNCHES:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv python bench.py --workload ${LAUNCH_W:-c4} --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep > $O/ncu_launch.log 2>&1
python tools/launch_summary.py $O/launches_c4.csv 2>/dev/null | head -12
fi
