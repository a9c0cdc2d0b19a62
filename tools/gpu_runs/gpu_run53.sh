# compute-sanitizer (memcheck / racecheck / synccheck) over every kernel family at the current build.
mkdir -p gpurun_out
{ echo "# compute-sanitizer over every kernel family (tools/sanitize_target.py), B200, round 1, final build"
  for tool in memcheck racecheck synccheck; do echo "== $tool"; timeout 1200 compute-sanitizer --tool $tool python tools/sanitize_target.py 2>&1 | grep -E "sanitize target|ERROR SUMMARY|RACECHECK SUMMARY|Error|error" | head -8; done; } > gpurun_out/r53_sanitizer.txt 2>&1
cat gpurun_out/r53_sanitizer.txt
