# Round 2 pass 8: gaussian/lognormal variants (fp64-derived centred tables, lognormal ulps).
mkdir -p gpurun_out
timeout 900 ./tools/bm_variants > gpurun_out/r2_8_bm_variants.txt 2>&1
cat gpurun_out/r2_8_bm_variants.txt
