# MRG segmented-rows layout: full GPU suite, then A/B against the previous per-lane-run layout (var_old) and a 5-CTA bound.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -8 > gpurun_out/r26_pytest.txt
cat gpurun_out/r26_pytest.txt
python tools/ab_lib.py mrg_f64 28 3 old main b5 > gpurun_out/r26_ab.txt 2>&1
python tools/ab_lib.py mrg_bits 28 3 old main b5 >> gpurun_out/r26_ab.txt 2>&1
python tools/ab_lib.py mrg_f64 30 2 old main >> gpurun_out/r26_ab.txt 2>&1
cat gpurun_out/r26_ab.txt
