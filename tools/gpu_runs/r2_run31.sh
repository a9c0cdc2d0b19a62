# Round 2 pass 31: C5 end-to-end vs pipeline chunk size.
mkdir -p gpurun_out
for c in 512 1024 2048 4096; do
  timeout 600 python bench.py --workload c5_full --steps 15 --warmup 3 --no-cpu --c5-chunk $c > gpurun_out/r2_31_c5_$c.json 2> gpurun_out/r2_31_c5_$c.err
  echo "chunk $c: $(grep 'step ms' gpurun_out/r2_31_c5_$c.err)"
done
