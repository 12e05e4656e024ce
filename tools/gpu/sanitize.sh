# compute-sanitizer over every hand-written kernel family (tools/sanitize_small.py)
set -x
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -5 gpurun_out/sanitize_$tool.log
done
