# A/B: I2FP-free unit conversion mixes for the headline kernel.
mkdir -p gpurun_out
python tools/ab_lib.py unit_f32 32 3 m0 m1 m3 m5 m7 m15 > gpurun_out/r17_ab_unit_2p32.txt 2>&1
python tools/ab_lib.py unit_f32 30 3 m0 m5 m15 > gpurun_out/r17_ab_unit_2p30.txt 2>&1
cat gpurun_out/r17_ab_unit_*.txt
