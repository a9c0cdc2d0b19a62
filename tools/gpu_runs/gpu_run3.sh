mkdir -p gpurun_out
./tools/philox_variants > gpurun_out/r3_variants.txt 2>&1
cat gpurun_out/r3_variants.txt
