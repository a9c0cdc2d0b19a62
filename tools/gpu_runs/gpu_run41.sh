# Lognormal: table scaled by s*sqrt(2 ln 2)*log2(e), ex2 of one FMA: A/B vs HEAD, accuracy, GPU suite.
mkdir -p gpurun_out
python tools/ab_lib.py logn_f32 30 3 old main > gpurun_out/r41_ab.txt 2>&1
python tools/ab_acc.py main >> gpurun_out/r41_ab.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1 >> gpurun_out/r41_ab.txt
timeout 300 python bench.py --workload c3_logn --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r41_c3_logn.json 2>gpurun_out/r41_c3_logn.err
cat gpurun_out/r41_ab.txt; python -c "import json; d=json.load(open('gpurun_out/r41_c3_logn.json')); print(d['value'], d['roofline']['frac'])"
