# Round 2 pass 73: final validation at HEAD (after the normalisation rewrite, deposit robustness, C5 host path) -- full GPU suite, smoke, default bench, reference arm,
# launch list of the default bench command, headline ncu summary, sanitizer.
mkdir -p gpurun_out /tmp/ncu
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -4 > gpurun_out/r2_73_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_73_smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2_73_c4.json 2> gpurun_out/r2_73_c4.err
timeout 600 python bench.py --impl reference > gpurun_out/r2_73_reference.json 2> gpurun_out/r2_73_reference.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bench_c4.csv python bench.py > gpurun_out/r2_73_bench_under_ncu.json 2> gpurun_out/r2_73_bench_under_ncu.err
python tools/launch_share.py gpurun_out/r2_launches_bench_c4.csv > gpurun_out/r2_73_launch_share_c4.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"philox_kernel" -c 1 -s 1 -o /tmp/ncu/head python tools/ncu_target.py unit_f32 32 3 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/ncu/head.ncu-rep > gpurun_out/r2_73_ncu_unit_f32_2p32.txt 2>&1
rm -f gpurun_out/sanitizer.txt; bash tools/sanitize.sh > /dev/null 2>&1
cat gpurun_out/r2_73_pytest.txt gpurun_out/r2_73_smoke.txt gpurun_out/r2_73_launch_share_c4.txt gpurun_out/sanitizer.txt
python -c "
import json
for f in ('gpurun_out/r2_73_c4.json','gpurun_out/r2_73_reference.json'):
    d=json.loads(open(f).read().strip().splitlines()[-1]); r=d.get('roofline') or {}
    print(f, d['value'], r.get('frac'), r.get('frac_of_fill'), (d.get('e2e') or {}).get('value'), json.dumps(d.get('e2e_reference_seam'))[:200], json.dumps(d.get('clocks'))[:150])
"
head -8 gpurun_out/r2_73_ncu_unit_f32_2p32.txt
