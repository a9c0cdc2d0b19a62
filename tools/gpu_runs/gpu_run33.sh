# C5 array planning: calosim GPU tests (golden + chunking), C5 full bench, host profile.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_calosim.py -x -q 2>&1 | tail -3 > gpurun_out/r33_pytest.txt
cat gpurun_out/r33_pytest.txt
timeout 600 python bench.py --workload c5_full --steps 5 --warmup 1 > gpurun_out/r33_c5_full.json 2> gpurun_out/r33_c5_full.err
cat gpurun_out/r33_c5_full.json
python tools/c5_profile.py > gpurun_out/r33_c5prof.txt 2>&1; head -30 gpurun_out/r33_c5prof.txt
