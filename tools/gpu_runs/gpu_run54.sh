# ncu --set full of the exact fp32 gaussian and the fp64 gaussian (2^28).
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:philox -c 1 -s 2 -o gpurun_out/r54_exact python tools/ncu_target.py gauss_f32_exact 28 3 > gpurun_out/r54_ncu_exact.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:philox -c 1 -s 1 -o gpurun_out/r54_g64 python tools/ncu_target.py gauss_f64 28 2 > gpurun_out/r54_ncu_g64.log 2>&1
ls -la gpurun_out/r54_*.ncu-rep; tail -3 gpurun_out/r54_ncu_exact.log
