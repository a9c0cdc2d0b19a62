# Round 2 pass 32: CTA residency of the persistent Philox kernels (PRNG_TRACE_CTA build).
mkdir -p gpurun_out
export PRNG_B200_LIB=$PWD/build/var_trace/libprng_b200.so
for spec in "unit_f32 32" "unit_f32 30" "bits 32" "gauss_f32 30" "unit_f32 24"; do
  set -- $spec
  timeout 300 python tools/cta_residency.py $1 $2 2>&1 | tail -4
done | tee gpurun_out/r2_32_cta_residency.txt
