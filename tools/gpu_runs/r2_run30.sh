# Round 2 pass 30: unit fp32 conversion with the 2^-24 scaling on the exponent bits (ALU) vs FMUL.
mkdir -p gpurun_out
cd tools
timeout 900 python ab_lib.py unit_f32 32 4 main is1 is2 > ../gpurun_out/r2_30_ab_unit32.txt 2>&1
timeout 600 python ab_lib.py unit_f32 30 4 main is1 is2 > ../gpurun_out/r2_30_ab_unit30.txt 2>&1
cd ..
cat gpurun_out/r2_30_ab_unit32.txt gpurun_out/r2_30_ab_unit30.txt
