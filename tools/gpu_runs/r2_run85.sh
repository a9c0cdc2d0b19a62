# Round 2 pass 85: exact fp32 gaussian with an rsqrt + Newton sqrt on its uncorrected path (bound measured with the tables).
mkdir -p gpurun_out
export PRNG_B200_LIB=$PWD/build/var_fsq/libprng_b200.so
timeout 1200 python -m pytest tests/test_exact_gaussian.py "tests/test_gpu_parity.py::test_box_muller_exhaustive_24bit" -q -m gpu -s 2>&1 | grep -E "passed|failed|exact_bounds|Error" | tail -5
unset PRNG_B200_LIB
cd tools
timeout 900 python ab_lib.py gauss_f32_exact 30 3 main fsq > ../gpurun_out/r2_85_ab_exact.txt 2>&1
cd ..
cat gpurun_out/r2_85_ab_exact.txt
