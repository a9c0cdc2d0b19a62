# Round 2 pass 7: non-persistent Philox kernels + gaussian variants incl. non-persistent.
mkdir -p gpurun_out
timeout 600 ./tools/philox_np > gpurun_out/r2_7_philox_np.txt 2>&1
timeout 900 ./tools/bm_variants > gpurun_out/r2_7_bm_variants.txt 2>&1
cat gpurun_out/r2_7_philox_np.txt gpurun_out/r2_7_bm_variants.txt
