# compute-sanitizer over every kernel family (small sizes); summary to gpurun_out/sanitizer.txt
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  echo "== $tool" >> gpurun_out/sanitizer.txt
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_target.py 2>&1 | \
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Race|Hazard|sanitize target" >> gpurun_out/sanitizer.txt
done
cat gpurun_out/sanitizer.txt
