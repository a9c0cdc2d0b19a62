# Final refresh at HEAD: full GPU suite, smoke, every bench line, reference arm, launch list of the headline command.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/r52_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r52_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r52_c4.json 2> gpurun_out/r52_c4.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r52_reference.json 2>/dev/null
for w in c1 c2 c3_gauss c3_logn c4_bits; do timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r52_$w.json 2>gpurun_out/r52_$w.err; done
timeout 600 python bench.py --workload c5 --steps 10 --warmup 2 > gpurun_out/r52_c5.json 2>gpurun_out/r52_c5.err
timeout 600 python bench.py --workload c5_full --steps 10 --warmup 2 > gpurun_out/r52_c5_full.json 2>gpurun_out/r52_c5_full.err
timeout 900 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --sweep > gpurun_out/r52_sweep.json 2>gpurun_out/r52_sweep.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r52_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
cat gpurun_out/r52_pytest.txt gpurun_out/r52_smoke.txt
for f in gpurun_out/r52_*.json; do echo "$f"; python -c "import json,sys; d=json.load(open('$f')); print(d.get('value'), d.get('roofline',{}).get('frac') if d.get('roofline') else '', d.get('clocks'))"; done
