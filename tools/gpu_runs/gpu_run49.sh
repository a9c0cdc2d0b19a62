# ncu --set full of the headline kernel (2^32, current build) and the fast gaussian (2^30); summaries + opcode stalls.
mkdir -p gpurun_out
timeout 400 ncu --set full --clock-control none --import-source on -k regex:philox -c 1 -s 1 -o gpurun_out/r49_c4 python tools/ncu_target.py unit_f32 32 2 > gpurun_out/r49_ncu_c4.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:philox -c 1 -s 1 -o gpurun_out/r49_gauss python tools/ncu_target.py gauss_f32 30 2 > gpurun_out/r49_ncu_gauss.log 2>&1
ls -la gpurun_out/r49_*.ncu-rep
