# Round 2 pass 18 (fresh container): full GPU suite + smoke + default bench at HEAD,
# launch list of the default bench command, one --set full capture per bench kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/r2_18_gpu.txt 2>&1
lscpu | head -20 >> gpurun_out/r2_18_gpu.txt
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -8 > gpurun_out/r2_18_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_18_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r2_18_bench.json 2> gpurun_out/r2_18_bench.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bench_c4.csv python bench.py > gpurun_out/r2_18_bench_under_ncu.json 2> gpurun_out/r2_18_bench_under_ncu.err
for spec in "unit_f32 32" "bits 32" "gauss_f32 30" "logn_f32 30" "gauss_f32_exact 30" "mrg_f64 28" "mrg_bits 28"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mrg_kernel|philox_kernel" -c 1 -s 1 -o gpurun_out/r2_ncu_$1_2p$2 python tools/ncu_target.py $1 $2 3 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/r2_ncu_$1_2p$2.ncu-rep > gpurun_out/r2_ncu_$1_2p$2.txt 2>&1
done
python tools/launch_share.py gpurun_out/r2_launches_bench_c4.csv > gpurun_out/r2_launches_share.txt 2>&1
cat gpurun_out/r2_18_pytest.txt gpurun_out/r2_18_smoke.txt gpurun_out/r2_launches_share.txt
head -c 600 gpurun_out/r2_18_bench.json
for f in gpurun_out/r2_ncu_*.txt; do echo "== $f"; head -12 $f; done
