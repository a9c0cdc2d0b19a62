set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/r2_pytest_gpu.txt
for w in bits unit_f32 fill; do
  timeout 300 ncu --set full --clock-control none --import-source on -c 1 -s 1 -o gpurun_out/r2_$w python tools/ncu_target.py $w 28 3 > gpurun_out/r2_ncu_$w.log 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:philox -c 1 -s 1 -o gpurun_out/r2_gauss_f32 python tools/ncu_target.py gauss_f32 28 3 > gpurun_out/r2_ncu_gauss.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:mrg -c 1 -s 1 -o gpurun_out/r2_mrg_f64 python tools/ncu_target.py mrg_f64 28 3 > gpurun_out/r2_ncu_mrg.log 2>&1
cat gpurun_out/r2_pytest_gpu.txt
ls -la gpurun_out
