# C2 / C3 bench lines with their CPU baselines (reference core on the host cores).
mkdir -p gpurun_out
for w in c2 c3_gauss; do timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e > gpurun_out/r62_$w.json 2>gpurun_out/r62_$w.err; python -c "import json; d=json.load(open('gpurun_out/r62_$w.json')); print('$w', d['value'], d['roofline']['frac'], d['cpu_baseline'])"; done
