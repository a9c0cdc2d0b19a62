# HEAD check: GPU suite, smoke, headline bench and reference arm as the driver runs them.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1 > gpurun_out/r59_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r59_smoke.txt 2>&1
timeout 600 python bench.py --gpus 1 --steps 50 --warmup 5 > gpurun_out/r59_c4.json 2> gpurun_out/r59_c4.err
timeout 300 python bench.py --impl reference --gpus 1 --steps 5 --warmup 3 > gpurun_out/r59_reference.json 2>/dev/null
cat gpurun_out/r59_pytest.txt gpurun_out/r59_smoke.txt gpurun_out/r59_c4.json gpurun_out/r59_reference.json
