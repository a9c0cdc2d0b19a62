mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -25 > gpurun_out/r4_pytest_gpu.txt
timeout 600 python tools/probe.py > gpurun_out/r4_probe.txt 2>&1
cat gpurun_out/r4_pytest_gpu.txt gpurun_out/r4_probe.txt
