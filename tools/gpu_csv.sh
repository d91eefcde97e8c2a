#!/bin/bash
# GPU check of the points-CSV reader, then the whole GPU suite.
mkdir -p gpurun_out/csv
python -m pytest tests/test_csv.py tests/test_cpp_api.py -m gpu -x -q -s > gpurun_out/csv/csv_tests.log 2>&1
echo "csv rc=$?"
tail -5 gpurun_out/csv/csv_tests.log
python -m pytest tests -m gpu -x -q > gpurun_out/csv/gpu_all.log 2>&1
echo "all rc=$?"
tail -3 gpurun_out/csv/gpu_all.log
