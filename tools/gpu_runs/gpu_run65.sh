# Final HEAD validation: GPU suite, smoke, headline, reference arm, C3 lines (+ CPU baselines), sanitizer on the new lognormal instantiation.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1 > gpurun_out/r65_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r65_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r65_c4.json 2> gpurun_out/r65_c4.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r65_reference.json 2>/dev/null
for w in c3_gauss c3_logn; do timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e > gpurun_out/r65_$w.json 2>gpurun_out/r65_$w.err; done
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_target.py 2>&1 | grep -E "sanitize target|ERROR SUMMARY" > gpurun_out/r65_memcheck.txt
cat gpurun_out/r65_pytest.txt gpurun_out/r65_smoke.txt gpurun_out/r65_memcheck.txt
for f in gpurun_out/r65_c4.json gpurun_out/r65_c3_gauss.json gpurun_out/r65_c3_logn.json gpurun_out/r65_reference.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['value'], (d.get('roofline') or {}).get('frac'), (d.get('cpu_baseline') or {}).get('value'))"; done
