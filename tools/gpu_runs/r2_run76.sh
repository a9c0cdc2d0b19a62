# Round 2 pass 76: deposit buckets aliasing the bitmap (56 KB, 4 CTAs/SM) vs the committed layout.
mkdir -p gpurun_out
PRNG_B200_LIB=$PWD/build/var_da/libprng_b200.so timeout 600 python -m pytest tests/test_calo_deposit.py tests/test_calosim.py -q -m gpu 2>&1 | tail -2
bash tools/c5_dep_ab.sh main da main da | tee gpurun_out/r2_76_dep_ab.txt
