# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py
# (every kernel family and mode); summaries under gpurun_out/sanitize_*.log
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 300 python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_plain.log
for tool in memcheck racecheck synccheck; do
  extra=""; [ $tool = memcheck ] && extra="--leak-check no"
  timeout 2400 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -3 gpurun_out/sanitize_$tool.log
done
echo done
