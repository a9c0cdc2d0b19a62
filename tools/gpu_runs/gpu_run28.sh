# Software-pipelined Philox + fast Box-Muller: A/B of register bounds vs the unpipelined loop.
mkdir -p gpurun_out
python tools/ab_lib.py gauss_f32 30 3 nopipe main pb5 pb4 > gpurun_out/r28_ab.txt 2>&1
python tools/ab_lib.py logn_f32 30 3 nopipe main pb5 pb4 >> gpurun_out/r28_ab.txt 2>&1
cat gpurun_out/r28_ab.txt
