# Round 2 pass 35: first exact request under CUDA-graph capture; bench with the fill_ ceiling keys.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_exact_gaussian.py -q -m gpu -k capture 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --warmup 3 --no-e2e --no-plugin-e2e --no-cpu > gpurun_out/r2_35_c4.json 2> gpurun_out/r2_35_c4.err
python -c "
import json; d=json.loads(open('gpurun_out/r2_35_c4.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], r['frac'], r['frac_of_write_peak'], r['frac_of_fill'], r['frac_of_nominal_8tbs'], r['write_peak'])"
