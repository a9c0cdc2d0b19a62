# Round 2 pass 63: fast gaussian / lognormal kernels with a 6-CTA (40-register) bound.
mkdir -p gpurun_out
cd tools
timeout 900 python ab_lib.py gauss_f32 30 4 main gm6 gm5 > ../gpurun_out/r2_63_ab_gauss.txt 2>&1
timeout 900 python ab_lib.py logn_f32 30 4 main gm6 > ../gpurun_out/r2_63_ab_logn.txt 2>&1
cd ..
cat gpurun_out/r2_63_ab_*.txt
