# Round 2 pass 24: full GPU suite + compute-sanitizer (memcheck/racecheck/synccheck) on the CUB-free deposit build.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4 > gpurun_out/r2_24_pytest.txt
cat gpurun_out/r2_24_pytest.txt
rm -f gpurun_out/sanitizer.txt
bash tools/sanitize.sh
