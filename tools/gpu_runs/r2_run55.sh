# Round 2 pass 55: XU conversion with the 6-CTA register bound; ncu pipes of the xu variant.
mkdir -p gpurun_out /tmp/ncu
cd tools
timeout 900 python ab_lib.py unit_f32 32 4 main xu6 xu > ../gpurun_out/r2_55_ab_unit32.txt 2>&1
cd ..
cat gpurun_out/r2_55_ab_unit32.txt
PRNG_B200_LIB=$PWD/build/var_xu/libprng_b200.so timeout 600 ncu --set full --clock-control none -k regex:philox_kernel -c 1 -s 1 -o /tmp/ncu/xu python tools/ncu_target.py unit_f32 32 3 > /dev/null 2>&1
python tools/ncu_summary.py /tmp/ncu/xu.ncu-rep
