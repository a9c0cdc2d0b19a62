# MRG plan: segmented rows for plain fp64 (5-CTA bound), per-lane runs otherwise; full GPU suite + A/B vs previous layout.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3 > gpurun_out/r27_pytest.txt
cat gpurun_out/r27_pytest.txt
python tools/ab_lib.py mrg_f64 28 3 old main > gpurun_out/r27_ab.txt 2>&1
python tools/ab_lib.py mrg_bits 28 3 old main >> gpurun_out/r27_ab.txt 2>&1
python tools/ab_lib.py mrg_f64 30 2 old main >> gpurun_out/r27_ab.txt 2>&1
timeout 300 python bench.py --workload c2 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r27_c2.json 2>gpurun_out/r27_c2.err
cat gpurun_out/r27_ab.txt gpurun_out/r27_c2.json
