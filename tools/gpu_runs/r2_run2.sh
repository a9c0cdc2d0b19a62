# Round 2 pass 2: full GPU suite after the tolerance-import and subnormal-test fixes,
# default bench, --gpus 2 self-launch, C3 lines.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/r2_2_pytest.txt
timeout 600 python bench.py > gpurun_out/r2_2_c4.json 2> gpurun_out/r2_2_c4.err
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2_2_g2.json 2> gpurun_out/r2_2_g2.err
timeout 600 python bench.py --workload c3_gauss --steps 20 --warmup 3 --no-e2e > gpurun_out/r2_2_c3g.json 2> gpurun_out/r2_2_c3g.err
timeout 600 python bench.py --workload c3_logn --steps 20 --warmup 3 --no-e2e > gpurun_out/r2_2_c3l.json 2> gpurun_out/r2_2_c3l.err
tail -3 gpurun_out/r2_2_pytest.txt
for f in c4 g2 c3g c3l; do echo "== $f"; tail -c 2500 gpurun_out/r2_2_$f.json; grep -i "error" gpurun_out/r2_2_$f.err | tail -3; done
