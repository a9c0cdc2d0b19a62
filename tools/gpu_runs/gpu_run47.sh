# Philox round keys as precomputed kernel-parameter operands (main) vs recomputed in the loop (old = previous HEAD).
mkdir -p gpurun_out
python tools/ab_lib.py unit_f32 32 3 old main > gpurun_out/r47_ab.txt 2>&1
python tools/ab_lib.py unit_f32 30 3 old main >> gpurun_out/r47_ab.txt 2>&1
python tools/ab_lib.py bits 32 3 old main >> gpurun_out/r47_ab.txt 2>&1
python tools/ab_lib.py gauss_f32 30 3 old main >> gpurun_out/r47_ab.txt 2>&1
python tools/ab_lib.py logn_f32 30 3 old main >> gpurun_out/r47_ab.txt 2>&1
python tools/ab_lib.py unit_f64 31 3 old main >> gpurun_out/r47_ab.txt 2>&1
cat gpurun_out/r47_ab.txt
