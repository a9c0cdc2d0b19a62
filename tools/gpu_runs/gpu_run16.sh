# ncu --set full (with source) of the headline kernel and the C2/C3 kernels; opcode stall attribution.
mkdir -p gpurun_out
for w in unit_f32 mrg_f64 gauss_f32 logn_f32; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"mrg|philox" -c 1 -s 1 -o gpurun_out/r16_$w python tools/ncu_target.py $w 28 3 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/r16_$w.ncu-rep > gpurun_out/r16_$w.txt 2>&1
  python tools/ncu_opcodes.py gpurun_out/r16_$w.ncu-rep >> gpurun_out/r16_$w.txt 2>&1
  ncu -i gpurun_out/r16_$w.ncu-rep --page source --csv --print-source sass > gpurun_out/r16_${w}_src.csv 2>/dev/null
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"philox" -c 1 -s 1 -o gpurun_out/r16_c4_2p32 python tools/ncu_target.py unit_f32 32 2 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r16_c4_2p32.ncu-rep > gpurun_out/r16_c4_2p32.txt 2>&1
rm -f gpurun_out/r16_c4_2p32.ncu-rep gpurun_out/r16_logn_f32.ncu-rep
du -sh gpurun_out/*
cat gpurun_out/r16_*.txt
