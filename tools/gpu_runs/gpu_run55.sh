# Exact gaussian: correction gathers issued one pass ahead (pipelined loop); register bounds; bit-identity via hashes + GPU suite.
mkdir -p gpurun_out
python tools/ab_lib.py gauss_f32_exact 28 3 old main eb3 eb4 > gpurun_out/r55_ab.txt 2>&1
python tools/ab_lib.py gauss_f64_exact 28 3 old main eb3 eb4 >> gpurun_out/r55_ab.txt 2>&1
cat gpurun_out/r55_ab.txt
timeout 900 python -m pytest tests -q -m gpu -k "exact" 2>&1 | tail -1
