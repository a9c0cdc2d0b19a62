mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/r7_pytest.txt
timeout 600 python bench.py --workload c5 --steps 10 > gpurun_out/r7_c5.json 2> gpurun_out/r7_c5.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --sweep > gpurun_out/r7_sweep.json 2> gpurun_out/r7_sweep.err
for w in c2 c3_gauss c3_logn c4_bits c1; do timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r7_$w.json 2>gpurun_out/r7_$w.err; done
cat gpurun_out/r7_pytest.txt gpurun_out/r7_c5.json; tail -3 gpurun_out/r7_c5.err; grep sweep gpurun_out/r7_sweep.err | head -40
for w in c2 c3_gauss c3_logn c4_bits c1; do python -c "import json;d=json.load(open('gpurun_out/r7_$w.json'));print('$w', round(d['value'],1), d['unit'], round(d['roofline']['achieved']), round(d['roofline']['frac'],3))"; done
