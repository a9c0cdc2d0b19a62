# Box-Muller instruction trims (scaled series on kf, single-LOP3 mantissa): bit-identity + speed vs previous HEAD lib (old),
# and the table-scaled variant (tabs): speed + exhaustive accuracy.
mkdir -p gpurun_out
python tools/ab_lib.py gauss_f32 30 3 old main tabs > gpurun_out/r39_ab.txt 2>&1
python tools/ab_lib.py logn_f32 30 3 old main tabs >> gpurun_out/r39_ab.txt 2>&1
python tools/ab_acc.py main tabs >> gpurun_out/r39_ab.txt 2>&1
cat gpurun_out/r39_ab.txt
