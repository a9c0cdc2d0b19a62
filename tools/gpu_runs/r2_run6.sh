# Round 2 pass 6: non-persistent Philox kernels (tools/philox_np.cu) and the fast
# Box-Muller design study (tools/bm_variants.cu: throughput + exhaustive ulps).
mkdir -p gpurun_out
timeout 600 ./tools/philox_np > gpurun_out/r2_6_philox_np.txt 2>&1
timeout 900 ./tools/bm_variants > gpurun_out/r2_6_bm_variants.txt 2>&1
cat gpurun_out/r2_6_philox_np.txt gpurun_out/r2_6_bm_variants.txt
