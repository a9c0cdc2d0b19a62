# Round 2 pass 37: C5 critical path parts (D2H alone, host profile).
mkdir -p gpurun_out
timeout 600 python tools/c5_parts.py 2>&1 | tee gpurun_out/r2_37_c5_parts.txt | head -60
