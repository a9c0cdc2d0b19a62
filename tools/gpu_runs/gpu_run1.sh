set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)"; free -g | head -2
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -30 > gpurun_out/r1_pytest_gpu.txt
timeout 600 python tools/probe.py > gpurun_out/r1_probe.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
cat gpurun_out/r1_pytest_gpu.txt gpurun_out/r1_probe.txt gpurun_out/r1_bench.json; tail -5 gpurun_out/r1_bench.err
