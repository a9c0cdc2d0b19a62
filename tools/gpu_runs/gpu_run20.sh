# GPU suite on the new fast Box-Muller; MRG occupancy/chain A/B.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 > gpurun_out/r20_pytest.txt
python tools/ab_lib.py mrg_f64 28 3 main r4c2 r5c2 r8c1 r12c1 > gpurun_out/r20_ab_mrg_f64.txt 2>&1
python tools/ab_lib.py mrg_bits 28 2 main r5c2 r8c1 r12c1 > gpurun_out/r20_ab_mrg_bits.txt 2>&1
cat gpurun_out/r20_*.txt
