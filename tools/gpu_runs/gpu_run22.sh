# Session-4 (re-created container) verification of HEAD: tests, smoke, headline, reference arm, C2/C3 lines.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/r22_smi.txt
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -8 > gpurun_out/r22_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r22_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r22_c4.json 2> gpurun_out/r22_c4.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r22_reference.json 2>gpurun_out/r22_reference.err
for w in c2 c3_gauss c3_logn; do timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r22_$w.json 2>gpurun_out/r22_$w.err; done
cat gpurun_out/r22_pytest.txt gpurun_out/r22_smoke.txt gpurun_out/r22_c4.json gpurun_out/r22_reference.json gpurun_out/r22_c2.json gpurun_out/r22_c3_*.json
