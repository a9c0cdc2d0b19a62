# MRG kernel with per-transform chain arrays, 4-CTA bound for the segmented fp64 path: GPU suite, C2 bench, ncu.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1 > gpurun_out/r45_pytest.txt
cat gpurun_out/r45_pytest.txt
timeout 300 python bench.py --workload c2 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r45_c2.json 2>gpurun_out/r45_c2.err
python -c "import json; d=json.load(open('gpurun_out/r45_c2.json')); print('c2', d['value'], d['roofline']['frac'])"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:mrg -c 1 -s 1 -o gpurun_out/r45_c2 python tools/ncu_target.py mrg_f64 28 2 > gpurun_out/r45_ncu_c2.log 2>&1
ncu -i gpurun_out/r45_c2.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active > gpurun_out/r45_c2_raw.csv 2>&1
cat gpurun_out/r45_c2_raw.csv
