# A/B round 2: fast Box-Muller table/series variants (timing + exhaustive accuracy).
mkdir -p gpurun_out
python tools/ab_lib.py gauss_f32 30 3 g0 main n1 n2 n3 n4 > gpurun_out/r19_ab_gauss.txt 2>&1
python tools/ab_lib.py logn_f32 30 2 g0 main n2 > gpurun_out/r19_ab_logn.txt 2>&1
python tools/ab_acc.py main n1 n2 n3 n4 > gpurun_out/r19_acc.txt 2>&1
cat gpurun_out/r19_*.txt
