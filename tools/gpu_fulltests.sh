#!/bin/bash
# the whole GPU suite (incl. full-size parity against golden_cache/) + smoke
cd ${GRAFT_REPO_ROOT:-.}
O=gpurun_out/fulltests; rm -rf $O; mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q --timeout 1800 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
