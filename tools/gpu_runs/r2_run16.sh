# Round 2 pass 16: full GPU suite on the current build (odd-element shifted stores,
# exact short forms), C3 lines incl. the odd-element case.
mkdir -p gpurun_out
rm -f gpurun_out/bm_ulp_bands.jsonl
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tail -8 > gpurun_out/r2_16_pytest.txt
for w in c3_gauss c3_logn c3_gauss_precise c3_gauss_exact c3_gauss_accurate; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e > gpurun_out/r2_16_$w.json 2> gpurun_out/r2_16_$w.err
done
timeout 600 python bench.py --workload c3_gauss --steps 20 --warmup 3 --no-e2e --out-offset 1 > gpurun_out/r2_16_c3_gauss_odd.json 2> gpurun_out/r2_16_c3_gauss_odd.err
cat gpurun_out/r2_16_pytest.txt
for w in c3_gauss c3_logn c3_gauss_precise c3_gauss_exact c3_gauss_accurate c3_gauss_odd; do python -c "
import json
try:
  d=json.loads(open('gpurun_out/r2_16_$w.json').read().strip().splitlines()[-1]); r=d['roofline']
  print('$w', round(d['value'],1), round(r['frac'],3), d['slice_check']['all_equal'], d['slice_check'].get('worst_err_over_allowed_rank0'))
except Exception as e: print('$w ERR', e)
"; done
