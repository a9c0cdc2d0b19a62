# Round 2 pass 9: centred fast Box-Muller in the library; loop / min-blocks A/B.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "box_muller or lognormal or gaussian or c3" 2>&1 | tail -15 > gpurun_out/r2_9_pytest.txt
cd tools
timeout 600 python ab_lib.py gauss_f32 30 3 main pipe1 m0 m5 > ../gpurun_out/r2_9_ab_gauss.txt 2>&1
timeout 600 python ab_lib.py logn_f32 30 3 main pipe1 m0 m5 > ../gpurun_out/r2_9_ab_logn.txt 2>&1
cd ..
cat gpurun_out/r2_9_pytest.txt gpurun_out/r2_9_ab_gauss.txt gpurun_out/r2_9_ab_logn.txt
