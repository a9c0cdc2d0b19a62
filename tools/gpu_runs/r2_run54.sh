# Round 2 pass 54: int->float conversion on the XU pipe (cvt.rm -> I2F.U32.RM) instead of I2FP (FMA-heavy).
mkdir -p gpurun_out
cd tools
timeout 900 python ab_lib.py unit_f32 32 4 main xu > ../gpurun_out/r2_54_ab_unit32.txt 2>&1
timeout 600 python ab_lib.py unit_f32 30 4 main xu > ../gpurun_out/r2_54_ab_unit30.txt 2>&1
timeout 600 python ab_lib.py uniform_f32 32 3 main xu > ../gpurun_out/r2_54_ab_uni32.txt 2>&1
timeout 600 python ab_lib.py gauss_f32 30 3 main xu xubm > ../gpurun_out/r2_54_ab_gauss.txt 2>&1
timeout 600 python ab_lib.py logn_f32 30 3 main xu xubm > ../gpurun_out/r2_54_ab_logn.txt 2>&1
cd ..
cat gpurun_out/r2_54_ab_*.txt
