# MRG layout edge-case full-array test; headline bench with the new clock sampler.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "segment_layout or mrg" 2>&1 | tail -3 > gpurun_out/r31_pytest.txt
cat gpurun_out/r31_pytest.txt
timeout 600 python bench.py > gpurun_out/r31_c4.json 2> gpurun_out/r31_c4.err
cat gpurun_out/r31_c4.json
