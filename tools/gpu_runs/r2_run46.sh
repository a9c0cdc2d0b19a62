# Round 2 pass 46: deposit register path with batched amount loads: 3 CTAs/SM (spills) vs 2 CTAs/SM.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_calo_deposit.py tests/test_calosim.py -x -q -m gpu 2>&1 | tail -2
bash tools/c5_dep_ab.sh main d2 | tee gpurun_out/r2_46_dep_ab.txt
