# A/B: fast fp32 Box-Muller variants (timing + exhaustive accuracy).
mkdir -p gpurun_out
python tools/ab_lib.py gauss_f32 30 3 g0 g1 g2 g3 g4 g6 > gpurun_out/r18_ab_gauss.txt 2>&1
python tools/ab_lib.py logn_f32 30 2 g0 g2 g3 g4 > gpurun_out/r18_ab_logn.txt 2>&1
python tools/ab_acc.py g0 g1 g2 g3 g4 g6 > gpurun_out/r18_acc.txt 2>&1
cat gpurun_out/r18_*.txt
