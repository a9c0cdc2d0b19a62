# Round 2 pass 52: wall time of the default bench command (driver contract: minutes).
mkdir -p gpurun_out
s=$(date +%s.%N); python bench.py > gpurun_out/r2_52_c4.json 2> gpurun_out/r2_52_c4.err; e=$(date +%s.%N)
echo "default bench wall s: $(python -c "print(round($e-$s,1))")"
s=$(date +%s.%N); python bench.py --steps 20 --warmup 3 > gpurun_out/r2_52_c4_20.json 2> gpurun_out/r2_52_c4_20.err; e=$(date +%s.%N)
echo "--steps 20 --warmup 3 wall s: $(python -c "print(round($e-$s,1))")"
cat gpurun_out/r2_52_c4.err | tail -8
free -g | head -2; nproc
