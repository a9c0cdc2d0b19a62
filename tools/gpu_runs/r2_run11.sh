# Round 2 pass 11: fp32 exact route with the rounding test (no gathers on the common path).
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -s -k "exact or lognormal_fast_dense or lognormal_param" 2>&1 | grep -E "route|exact_bounds|passed|failed|Error|assert" > gpurun_out/r2_11_pytest.txt
timeout 600 python bench.py --workload c3_gauss_exact --steps 20 --warmup 3 --no-e2e > gpurun_out/r2_11_c3_gauss_exact.json 2> gpurun_out/r2_11_c3_gauss_exact.err
cat gpurun_out/r2_11_pytest.txt
python -c "
import json
d=json.loads(open('gpurun_out/r2_11_c3_gauss_exact.json').read().strip().splitlines()[-1]); r=d['roofline']
print('exact', round(d['value'],1), round(r['frac'],3), d['slice_check'])"
tail -3 gpurun_out/r2_11_c3_gauss_exact.err
