#!/bin/bash
# CSV I/O on one B200: tests, tools/bench_csv.py, ncu of the parse and format kernels.
O=gpurun_out/csv
mkdir -p $O
python -m pytest tests/test_csv.py tests/test_cpp_api.py -m gpu -x -q > $O/tests.log 2>&1
echo "tests rc=$?"; tail -4 $O/tests.log
timeout 900 python tools/bench_csv.py --rows 10000000 > $O/bench.jsonl 2> $O/bench.err
rc=$?; echo "bench rc=$rc"; cut -c1-400 $O/bench.jsonl; tail -3 $O/bench.err
if [ $rc -eq 0 ]; then
  for k in csv_parse_kernel emit_format_kernel; do
    timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $O/full_$k \
       python tools/bench_csv.py --rows 10000000 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_$k.log 2>&1
    echo "ncu $k rc=$?"
  done
fi
