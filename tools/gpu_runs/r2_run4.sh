# Round 2 pass 4: odd-element pair bodies (PhiloxBody::mis), bench e2e check fix.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -5 > gpurun_out/r2_4_pytest.txt
timeout 600 python bench.py > gpurun_out/r2_4_c4.json 2> gpurun_out/r2_4_c4.err
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-e2e > gpurun_out/r2_4_g2.json 2> gpurun_out/r2_4_g2.err
timeout 600 python bench.py --workload c3_gauss --steps 20 --warmup 3 --no-e2e --out-offset 1 > gpurun_out/r2_4_c3g_odd.json 2> gpurun_out/r2_4_c3g_odd.err
timeout 600 python bench.py --workload c3_gauss --steps 20 --warmup 3 --no-e2e > gpurun_out/r2_4_c3g.json 2> gpurun_out/r2_4_c3g.err
tail -3 gpurun_out/r2_4_pytest.txt
for f in c4 g2 c3g_odd c3g; do echo "== $f"; python -c "
import json,sys
try:
  d=json.loads(open('gpurun_out/r2_4_$f.json').read().strip().splitlines()[-1])
  r=d['roofline']; print(d['value'], d['n_gpus'], r['frac'], r.get('frac_of_write_peak'), r.get('sustained_frac'), (d.get('e2e') or {}).get('value'), (d.get('slice_check') or {}).get('all_equal'), d['clocks'])
except Exception as e: print('ERR', e)
"; grep -i "error" gpurun_out/r2_4_$f.err | tail -3; done
