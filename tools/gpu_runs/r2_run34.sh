# Round 2 pass 34: C5 with a ramped chunk schedule (first chunk small, doubling to 2048).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_calosim.py -q -m gpu 2>&1 | tail -2
for f in 2048 1024 512 256 128 64; do
  timeout 600 python bench.py --workload c5_full --steps 15 --warmup 3 --no-cpu --c5-first $f > gpurun_out/r2_34_c5_$f.json 2> gpurun_out/r2_34_c5_$f.err
  echo "first $f: $(grep 'step ms' gpurun_out/r2_34_c5_$f.err)"
done
