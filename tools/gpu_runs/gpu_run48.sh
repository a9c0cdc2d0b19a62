# Round keys from the parameter table for the uniform transforms only: GPU suite, A/B vs previous HEAD, headline bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -1 > gpurun_out/r48_pytest.txt
cat gpurun_out/r48_pytest.txt
python tools/ab_lib.py unit_f32 30 4 old main > gpurun_out/r48_ab.txt 2>&1
python tools/ab_lib.py uniform_f32 30 3 old main >> gpurun_out/r48_ab.txt 2>&1
python tools/ab_lib.py bits 30 3 old main >> gpurun_out/r48_ab.txt 2>&1
python tools/ab_lib.py gauss_f32 30 2 old main >> gpurun_out/r48_ab.txt 2>&1
cat gpurun_out/r48_ab.txt
timeout 600 python bench.py > gpurun_out/r48_c4.json 2> gpurun_out/r48_c4.err
python -c "import json; d=json.load(open('gpurun_out/r48_c4.json')); print('c4', d['value'], d['roofline']['frac'], d['per_launch_ms'], d['clocks'])"
