# Round 2 pass 12: exact fp32 route with the integer-domain rounding test; unit conversion variants.
mkdir -p gpurun_out
timeout 900 ./tools/unit_conv > gpurun_out/r2_12_unit_conv.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -s -k "exact" 2>&1 | grep -E "route|exact_bounds|passed|failed|Error|assert" > gpurun_out/r2_12_pytest.txt
timeout 600 python bench.py --workload c3_gauss_exact --steps 20 --warmup 3 --no-e2e > gpurun_out/r2_12_c3_gauss_exact.json 2> gpurun_out/r2_12_c3_gauss_exact.err
cat gpurun_out/r2_12_unit_conv.txt gpurun_out/r2_12_pytest.txt
python -c "
import json
d=json.loads(open('gpurun_out/r2_12_c3_gauss_exact.json').read().strip().splitlines()[-1]); r=d['roofline']
print('exact', round(d['value'],1), round(r['frac'],3), d['slice_check']['all_equal'])"
tail -3 gpurun_out/r2_12_c3_gauss_exact.err
