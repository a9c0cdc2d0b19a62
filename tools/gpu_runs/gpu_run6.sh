mkdir -p gpurun_out
for w in mrg_bits gauss_f32 unit_f32; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"mrg|philox" -c 1 -s 1 -o gpurun_out/r6_$w python tools/ncu_target.py $w 28 3 > gpurun_out/r6_ncu_$w.log 2>&1
done
ls gpurun_out
