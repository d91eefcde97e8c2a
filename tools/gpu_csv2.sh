#!/bin/bash
# CSV reader v2 (single pass): tests, bench, ncu of the kernel.
mkdir -p gpurun_out/csv2
python -m pytest tests/test_csv.py tests/test_cpp_api.py -m gpu -x -q > gpurun_out/csv2/csv_tests.log 2>&1
echo "csv tests rc=$?"; tail -4 gpurun_out/csv2/csv_tests.log
timeout 600 python tools/bench_csv.py --rows 10000000 > gpurun_out/csv2/bench.json 2> gpurun_out/csv2/bench.err
rc=$?; echo "bench rc=$rc"; cat gpurun_out/csv2/bench.json; tail -3 gpurun_out/csv2/bench.err
if [ $rc -eq 0 ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:csv_parse_kernel -c 1 \
     -o gpurun_out/csv2/full_csv python tools/bench_csv.py --rows 10000000 --steps 1 --warmup 3 --no-cpu-baseline \
     > gpurun_out/csv2/ncu.log 2>&1
  echo "ncu rc=$?"
fi
python -m pytest tests -m gpu -x -q > gpurun_out/csv2/gpu_all.log 2>&1
echo "all rc=$?"; tail -2 gpurun_out/csv2/gpu_all.log
