# Round 2 pass 25: bench lines at HEAD (default C4 with e2e + plugin seam + cpu_baseline,
# C1, C2, C4 bits, C5 full, sweep, reference arm).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_25_c4.json 2> gpurun_out/r2_25_c4.err
timeout 600 python bench.py --impl reference > gpurun_out/r2_25_reference.json 2> gpurun_out/r2_25_reference.err
for w in c1 c2 c4_bits; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-plugin-e2e > gpurun_out/r2_25_$w.json 2> gpurun_out/r2_25_$w.err
done
timeout 600 python bench.py --workload c5_full --steps 10 --warmup 3 > gpurun_out/r2_25_c5_full.json 2> gpurun_out/r2_25_c5_full.err
timeout 900 python bench.py --sweep --steps 10 --warmup 3 --no-e2e --no-plugin-e2e --no-cpu > gpurun_out/r2_25_sweep.json 2> gpurun_out/r2_25_sweep.err
for f in gpurun_out/r2_25_*.json; do echo "== $f"; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
r=d.get('roofline') or {}
print(d.get('value'), d.get('unit'), 'frac', r.get('frac'), 'e2e', (d.get('e2e') or {}).get('value'), 'plugin', json.dumps(d.get('plugin_e2e'))[:200], 'cpu', (d.get('cpu_baseline') or {}).get('value'))
" 2>&1 | tail -2; done
tail -3 gpurun_out/r2_25_c4.err
