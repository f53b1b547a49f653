# compute-sanitizer over tools/sanitize_run.py, every tool
mkdir -p gpurun_out
for t in memcheck racecheck synccheck initcheck; do
  echo "== $t"
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_run.py 2>&1 | tail -4
  echo "exit ${PIPESTATUS[0]}"
done
