# Round 2 pass 3: bench lines after the slice_check fix; --gpus 2 self-launch test.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_robustness.py -q -m gpu 2>&1 | tail -5 > gpurun_out/r2_3_pytest.txt
timeout 600 python bench.py > gpurun_out/r2_3_c4.json 2> gpurun_out/r2_3_c4.err
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2_3_g2.json 2> gpurun_out/r2_3_g2.err
timeout 600 python bench.py --workload c3_gauss --steps 20 --warmup 3 --no-e2e > gpurun_out/r2_3_c3g.json 2> gpurun_out/r2_3_c3g.err
timeout 600 python bench.py --workload c3_logn --steps 20 --warmup 3 --no-e2e > gpurun_out/r2_3_c3l.json 2> gpurun_out/r2_3_c3l.err
timeout 600 python bench.py --workload c2 --steps 20 --warmup 3 --no-e2e > gpurun_out/r2_3_c2.json 2> gpurun_out/r2_3_c2.err
tail -3 gpurun_out/r2_3_pytest.txt
for f in c4 g2 c3g c3l c2; do echo "== $f"; python -c "
import json,sys
try:
  d=json.loads(open('gpurun_out/r2_3_$f.json').read().strip().splitlines()[-1])
  r=d['roofline']; print(d['value'], d['n_gpus'], r['frac'], r.get('frac_of_write_peak'), r.get('sustained_frac'), (d.get('e2e') or {}).get('value'), (d.get('slice_check') or {}).get('all_equal'), d['clocks'])
except Exception as e: print('ERR', e)
"; grep -i "error" gpurun_out/r2_3_$f.err | tail -3; done
