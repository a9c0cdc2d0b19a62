mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -s -k "exhaustive or golden or gauss or lane" 2>&1 | grep -E "max abs err|passed|failed|Error" | tail -12
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"philox" -c 1 -s 1 -o gpurun_out/r8_gauss_f64 python tools/ncu_target.py gauss_f64 26 3 > /dev/null 2>&1
python tools/probe.py 2>&1 | grep -E "gauss|logn"
