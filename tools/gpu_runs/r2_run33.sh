# Round 2 pass 33: dynamic chunk distribution (atomic counter) vs static grid-stride split.
mkdir -p gpurun_out
cd tools
timeout 900 python ab_lib.py unit_f32 32 3 main dw4 dw16 dw64 > ../gpurun_out/r2_33_ab_unit32.txt 2>&1
timeout 600 python ab_lib.py unit_f32 30 3 main dw4 dw16 dw64 > ../gpurun_out/r2_33_ab_unit30.txt 2>&1
timeout 600 python ab_lib.py bits 32 3 main dw16 > ../gpurun_out/r2_33_ab_bits32.txt 2>&1
timeout 600 python ab_lib.py unit_f32 24 3 main dw4 dw16 > ../gpurun_out/r2_33_ab_unit24.txt 2>&1
cd ..
cat gpurun_out/r2_33_ab_*.txt
