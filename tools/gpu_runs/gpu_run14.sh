# Round-1 refresh part B: ncu --set full captures (one launch each).
mkdir -p gpurun_out
for w in unit_f32 bits mrg_bits mrg_f64 gauss_f32 gauss_f64; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"mrg|philox" -c 1 -s 1 -o gpurun_out/r14_$w python tools/ncu_target.py $w 28 3 > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"philox" -c 1 -s 1 -o gpurun_out/r14_c4_2p32 python tools/ncu_target.py unit_f32 32 2 > /dev/null 2>&1
du -sh gpurun_out; ls -la gpurun_out
for f in gpurun_out/r14_*.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}.txt 2>&1; done
rm -f gpurun_out/r14_bits.ncu-rep gpurun_out/r14_gauss_f64.ncu-rep gpurun_out/r14_mrg_bits.ncu-rep gpurun_out/r14_mrg_f64.ncu-rep gpurun_out/r14_unit_f32.ncu-rep
du -sh gpurun_out
