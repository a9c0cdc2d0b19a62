# Round 2 pass 5: write-only store-pattern ceilings (tools/store_probe.cu), odd-offset gaussian line.
mkdir -p gpurun_out
timeout 300 ./tools/store_probe > gpurun_out/r2_5_store_probe.txt 2>&1
timeout 600 python bench.py --workload c3_gauss --steps 20 --warmup 3 --no-e2e --out-offset 1 > gpurun_out/r2_5_c3g_odd.json 2> gpurun_out/r2_5_c3g_odd.err
cat gpurun_out/r2_5_store_probe.txt
python -c "
import json
d=json.loads(open('gpurun_out/r2_5_c3g_odd.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['slice_check'])"
tail -2 gpurun_out/r2_5_c3g_odd.err
