# Round 2 pass 36: Philox round-1 product by 64-bit ALU adds across consecutive counters (ip1: uniform/bits; ip2: + fast gaussian).
mkdir -p gpurun_out
cd tools
timeout 900 python ab_lib.py unit_f32 32 4 main ip1 > ../gpurun_out/r2_36_ab_unit32.txt 2>&1
timeout 600 python ab_lib.py unit_f32 30 4 main ip1 > ../gpurun_out/r2_36_ab_unit30.txt 2>&1
timeout 600 python ab_lib.py bits 32 3 main ip1 > ../gpurun_out/r2_36_ab_bits32.txt 2>&1
timeout 600 python ab_lib.py unit_f64 31 3 main ip1 > ../gpurun_out/r2_36_ab_f64.txt 2>&1
timeout 600 python ab_lib.py uniform_f32 32 3 main ip1 > ../gpurun_out/r2_36_ab_uni32.txt 2>&1
timeout 600 python ab_lib.py gauss_f32 30 3 main ip2 > ../gpurun_out/r2_36_ab_gauss.txt 2>&1
cd ..
cat gpurun_out/r2_36_ab_*.txt
