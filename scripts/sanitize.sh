# compute-sanitizer over every kernel (scripts/sanitize_all.py): memcheck, racecheck, synccheck
set -u
mkdir -p gpurun_out
python scripts/sanitize_all.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/sanitize_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_all.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error" gpurun_out/sanitize_$tool.log | tail -4
done
