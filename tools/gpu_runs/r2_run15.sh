# Round 2 pass 15: exact fp32 route with short fp64 approximations on the common path.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -s -k "exact" 2>&1 | grep -E "exact_bounds|passed|failed|Error" > gpurun_out/r2_15_pytest.txt
cd tools
timeout 600 python ab_lib.py gauss_f32_exact 30 3 main full > ../gpurun_out/r2_15_ab_exact.txt 2>&1
timeout 600 python ab_lib.py gauss_f32_acc 30 3 main > ../gpurun_out/r2_15_ab_acc.txt 2>&1
cd ..
cat gpurun_out/r2_15_pytest.txt gpurun_out/r2_15_ab_exact.txt gpurun_out/r2_15_ab_acc.txt
