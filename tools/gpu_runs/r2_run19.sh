# Round 2 pass 19: CUB-free deposit kernel (tests + C5 bench + launch list),
# small-n grid A/B at 2^22/2^24, ncu --set full summaries of the bench kernels
# (reports moved out of gpurun_out: the 64 MiB copy-back limit).
mkdir -p gpurun_out /tmp/ncu
timeout 900 python -m pytest tests/test_calo_deposit.py tests/test_calosim.py -q -m gpu 2>&1 | tail -6 > gpurun_out/r2_19_pytest.txt
timeout 600 python bench.py --workload c5_full --steps 10 --warmup 3 > gpurun_out/r2_19_c5_full.json 2> gpurun_out/r2_19_c5_full.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c5_full.csv python bench.py --workload c5_full --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
python tools/launch_share.py gpurun_out/r2_launches_c5_full.csv > gpurun_out/r2_19_c5_share.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:calo_deposit -c 1 -o /tmp/ncu/dep python bench.py --workload c5_full --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py /tmp/ncu/dep.ncu-rep > gpurun_out/r2_ncu_calo_deposit.txt 2>&1
cd tools
for lg in 22 24 26; do timeout 600 python ab_lib.py unit_f32 $lg 3 main g2 g4 nc > ../gpurun_out/r2_19_ab_grid_$lg.txt 2>&1; done
cd ..
for spec in "unit_f32 32" "bits 32" "gauss_f32 30" "logn_f32 30" "gauss_f32_exact 30" "mrg_f64 28" "mrg_bits 28" "unit_f32 24"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mrg_kernel|philox_kernel" -c 1 -s 1 -o /tmp/ncu/r2_ncu_$1_2p$2 python tools/ncu_target.py $1 $2 3 > /dev/null 2>&1
  python tools/ncu_summary.py /tmp/ncu/r2_ncu_$1_2p$2.ncu-rep > gpurun_out/r2_ncu_$1_2p$2.txt 2>&1
  ncu -i /tmp/ncu/r2_ncu_$1_2p$2.ncu-rep --page source --csv --print-source sass 2>/dev/null | head -3000 > /tmp/ncu/src_$1_$2.csv
done
cp /tmp/ncu/r2_ncu_unit_f32_2p32.ncu-rep gpurun_out/ 2>/dev/null
du -sh gpurun_out
cat gpurun_out/r2_19_pytest.txt gpurun_out/r2_19_c5_share.txt gpurun_out/r2_ncu_calo_deposit.txt
head -c 1500 gpurun_out/r2_19_c5_full.json; echo
cat gpurun_out/r2_19_ab_grid_*.txt
