# Round 2 pass 13: exact fp32 route out-of-line fallback A/B, vs accurate on the same box.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -k "exact" 2>&1 | tail -2 > gpurun_out/r2_13_pytest.txt
cd tools
timeout 600 python ab_lib.py gauss_f32_exact 30 3 main inl > ../gpurun_out/r2_13_ab_exact.txt 2>&1
timeout 600 python ab_lib.py gauss_f32_acc 30 3 main > ../gpurun_out/r2_13_ab_acc.txt 2>&1
cd ..
cat gpurun_out/r2_13_pytest.txt gpurun_out/r2_13_ab_exact.txt gpurun_out/r2_13_ab_acc.txt
