# Pipelined fast Box-Muller (gauss 4-CTA bound) + MRG segmented rows: GPU suite, C2/C3 bench lines, ncu --set full of the new kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3 > gpurun_out/r29_pytest.txt
cat gpurun_out/r29_pytest.txt
for w in c2 c3_gauss c3_logn; do timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r29_$w.json 2>gpurun_out/r29_$w.err; done
for spec in "c2 mrg_f64 28" "c3_gauss gauss_f32 30" "c3_logn logn_f32 30"; do
  set -- $spec
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:"mrg|philox" -c 1 -s 1 -o gpurun_out/r29_$1 python tools/ncu_target.py $2 $3 2 > gpurun_out/r29_ncu_$1.log 2>&1
  ncu -i gpurun_out/r29_$1.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active > gpurun_out/r29_$1_raw.csv 2>&1
done
cat gpurun_out/r29_c*.json
