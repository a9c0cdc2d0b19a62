# Round 2, first GPU pass on the restored HEAD: GPU suite, smoke, default bench,
# reference arm, and the --gpus 2 self-launch (shared-GPU dry run on a 1-GPU box).
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r2_1_gpus.txt; lscpu | head -20 >> gpurun_out/r2_1_gpus.txt
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -30 > gpurun_out/r2_1_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_1_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r2_1_c4.json 2> gpurun_out/r2_1_c4.err
timeout 900 python bench.py --impl reference > gpurun_out/r2_1_ref.json 2> gpurun_out/r2_1_ref.err
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2_1_g2.json 2> gpurun_out/r2_1_g2.err
tail -3 gpurun_out/r2_1_pytest.txt; cat gpurun_out/r2_1_smoke.txt
for f in c4 ref g2; do echo "== $f"; tail -c 1500 gpurun_out/r2_1_$f.json; tail -3 gpurun_out/r2_1_$f.err; done
