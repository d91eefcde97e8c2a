#!/bin/bash
# The GPU test suite and the C++ drop-in API test on one B200.
mkdir -p gpurun_out/tests
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/tests/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/tests/pytest_gpu.log
