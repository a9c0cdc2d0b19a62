mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 | tee gpurun_out/r10_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py 2>gpurun_out/r10_bench.err | tee gpurun_out/r10_bench.json
timeout 600 python bench.py --workload c5_full --steps 3 --warmup 3 2>gpurun_out/r10_c5full.err | tee gpurun_out/r10_c5full.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1
