# Round 2 pass 51: normalisation with a depth-ordered node program.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_calosim.py tests/test_calo_deposit.py -q -m gpu 2>&1 | tail -2
timeout 600 python bench.py --workload c5_full --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_51_c5_full.json 2> gpurun_out/r2_51_c5_full.err
grep "step ms" gpurun_out/r2_51_c5_full.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c5_full.csv python bench.py --workload c5_full --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
python tools/launch_share.py gpurun_out/r2_launches_c5_full.csv
