# Box-Muller trims + gaussian table scaling: full GPU suite, accuracy, C3 bench lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2 > gpurun_out/r40_pytest.txt
cat gpurun_out/r40_pytest.txt
python tools/ab_acc.py main > gpurun_out/r40_acc.txt 2>&1; cat gpurun_out/r40_acc.txt
for w in c3_gauss c3_logn; do timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r40_$w.json 2>gpurun_out/r40_$w.err; python -c "import json; d=json.load(open('gpurun_out/r40_$w.json')); print('$w', d['value'], d['roofline']['frac'])"; done
