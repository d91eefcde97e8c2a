# compute-sanitizer is closed on this pool: run every kernel family under the
# checking build instead (device-side bounds / invariant traps, PC_DCHECK) --
# tools/sanitize_cases.py and the GPU parity suites -- plus the same cases on
# the release build.  Summaries: gpurun_out/devchecks_*.log
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 600 python tools/sanitize_cases.py > gpurun_out/devchecks_release.log 2>&1; echo "rc=$?" >> gpurun_out/devchecks_release.log
POLYCAST_LIB_VARIANT=debug timeout 900 python tools/sanitize_cases.py > gpurun_out/devchecks_cases.log 2>&1; echo "rc=$?" >> gpurun_out/devchecks_cases.log
POLYCAST_LIB_VARIANT=debug timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_full_parity.py tests/test_band_fuzz.py tests/test_csv.py -m gpu -q > gpurun_out/devchecks_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/devchecks_pytest.log
python - <<'PY'
import re
for f in ("release", "cases", "pytest"):
    t = open(f"gpurun_out/devchecks_{f}.log").read()
    print(f, "| PC_DCHECK failures:", t.count("PC_DCHECK failed"), "|", t.strip().splitlines()[-2:])
PY
