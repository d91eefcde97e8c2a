#!/bin/bash
# results-CSV writer: tests, CSV bench (reader + writer), ncu of the format kernel.
mkdir -p gpurun_out/emit
python -m pytest tests/test_csv.py tests/test_cpp_api.py -m gpu -x -q > gpurun_out/emit/tests.log 2>&1
echo "tests rc=$?"; tail -4 gpurun_out/emit/tests.log; grep -E "results:|csv:" gpurun_out/emit/tests.log
timeout 900 python tools/bench_csv.py --rows 10000000 > gpurun_out/emit/bench.jsonl 2> gpurun_out/emit/bench.err
rc=$?; echo "bench rc=$rc"; cut -c1-600 gpurun_out/emit/bench.jsonl; tail -3 gpurun_out/emit/bench.err
if [ $rc -eq 0 ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:emit_format_kernel -c 1 \
     -o gpurun_out/emit/full_emit python tools/bench_csv.py --rows 10000000 --steps 1 --warmup 3 --no-cpu-baseline \
     > gpurun_out/emit/ncu.log 2>&1
  echo "ncu rc=$?"
fi
python -m pytest tests -m gpu -x -q > gpurun_out/emit/gpu_all.log 2>&1
echo "all rc=$?"; tail -2 gpurun_out/emit/gpu_all.log
