# MRG fp64: start-state walk as exact fp64 split mat-vecs (main) vs integer folds (old): timing + MRG GPU tests.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -k "mrg or MRG or segment_layout" 2>&1 | tail -1 > gpurun_out/r69_pytest.txt
python tools/ab_lib.py mrg_f64 25 3 old main > gpurun_out/r69_ab.txt 2>&1
python tools/ab_lib.py mrg_f64 28 3 old main >> gpurun_out/r69_ab.txt 2>&1
python tools/ab_lib.py mrg_f64 30 2 old main >> gpurun_out/r69_ab.txt 2>&1
python tools/ab_lib.py mrg_bits 28 2 old main >> gpurun_out/r69_ab.txt 2>&1
cat gpurun_out/r69_pytest.txt gpurun_out/r69_ab.txt
