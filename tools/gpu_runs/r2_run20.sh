# Round 2 pass 20: deposit kernel with a double-buffered shared-memory walk.
mkdir -p gpurun_out /tmp/ncu
timeout 900 python -m pytest tests/test_calo_deposit.py tests/test_calosim.py -q -m gpu 2>&1 | tail -4 > gpurun_out/r2_20_pytest.txt
timeout 600 python bench.py --workload c5_full --steps 10 --warmup 3 --no-cpu > gpurun_out/r2_20_c5_full.json 2> gpurun_out/r2_20_c5_full.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c5_full.csv python bench.py --workload c5_full --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
python tools/launch_share.py gpurun_out/r2_launches_c5_full.csv > gpurun_out/r2_20_c5_share.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"calo_deposit|calo_normalize" -c 2 -o /tmp/ncu/dep python bench.py --workload c5_full --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py /tmp/ncu/dep.ncu-rep > gpurun_out/r2_ncu_calo_deposit.txt 2>&1
cat gpurun_out/r2_20_pytest.txt gpurun_out/r2_20_c5_share.txt gpurun_out/r2_ncu_calo_deposit.txt
head -c 700 gpurun_out/r2_20_c5_full.json; echo
