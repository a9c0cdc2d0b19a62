# Session-3 refresh: tests, smoke, headline bench, reference arm, launch list.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/r15_smi.txt
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 > gpurun_out/r15_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r15_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r15_c4.json 2> gpurun_out/r15_c4.err
timeout 600 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/r15_c4_b.json 2> gpurun_out/r15_c4_b.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r15_reference.json 2>/dev/null
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r15_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
cat gpurun_out/r15_pytest.txt gpurun_out/r15_smoke.txt gpurun_out/r15_c4.json gpurun_out/r15_c4_b.json
