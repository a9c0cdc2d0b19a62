# Final validation of HEAD: GPU suite, smoke, sanitizer memcheck, headline + C2 bench lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1 > gpurun_out/r70_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r70_smoke.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_target.py 2>&1 | grep -E "sanitize target|ERROR SUMMARY" > gpurun_out/r70_memcheck.txt
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_target.py 2>&1 | grep -E "sanitize target|RACECHECK SUMMARY" > gpurun_out/r70_racecheck.txt
timeout 600 python bench.py > gpurun_out/r70_c4.json 2> gpurun_out/r70_c4.err
timeout 600 python bench.py --workload c2 --steps 20 --warmup 3 --no-e2e > gpurun_out/r70_c2.json 2> gpurun_out/r70_c2.err
cat gpurun_out/r70_pytest.txt gpurun_out/r70_smoke.txt gpurun_out/r70_memcheck.txt gpurun_out/r70_racecheck.txt
for f in gpurun_out/r70_c4.json gpurun_out/r70_c2.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['value'], d['roofline']['frac'], d['cpu_baseline']['value'])"; done
