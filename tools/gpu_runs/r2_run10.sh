# Round 2 pass 10: centred fast + precise Box-Muller in the library: full GPU suite
# (exhaustive ulp bands), C3 bench lines, precise min-blocks A/B.
mkdir -p gpurun_out
rm -f gpurun_out/bm_ulp_bands.jsonl
timeout 1800 python -m pytest tests -q -m gpu -s -k "exhaustive or lognormal_fast_dense" 2>&1 | grep -E "route|passed|failed|Error|assert" > gpurun_out/r2_10_bands.txt
timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -8 > gpurun_out/r2_10_pytest.txt
for w in c3_gauss c3_logn c3_gauss_precise c3_logn_precise c3_gauss_exact; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e > gpurun_out/r2_10_$w.json 2> gpurun_out/r2_10_$w.err
done
cat gpurun_out/r2_10_bands.txt gpurun_out/r2_10_pytest.txt
for w in c3_gauss c3_logn c3_gauss_precise c3_logn_precise c3_gauss_exact; do python -c "
import json
try:
  d=json.loads(open('gpurun_out/r2_10_$w.json').read().strip().splitlines()[-1]); r=d['roofline']
  print('$w', round(d['value'],1), round(r['frac'],3), d['slice_check']['all_equal'], d['slice_check'].get('worst_err_over_allowed_rank0'))
except Exception as e: print('$w ERR', e)
"; done
