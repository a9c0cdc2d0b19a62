# Round 2 pass 39: register-resident deposit path for narrow-id events.
mkdir -p gpurun_out /tmp/ncu
timeout 900 python -m pytest tests/test_calo_deposit.py tests/test_calosim.py -q -m gpu 2>&1 | tail -4 > gpurun_out/r2_39_pytest.txt
cat gpurun_out/r2_39_pytest.txt
timeout 600 python bench.py --workload c5_full --steps 10 --warmup 3 > gpurun_out/r2_39_c5_full.json 2> gpurun_out/r2_39_c5_full.err
grep "step ms" gpurun_out/r2_39_c5_full.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c5_full.csv python bench.py --workload c5_full --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
python tools/launch_share.py gpurun_out/r2_launches_c5_full.csv
rm -f /tmp/ncu/dep6.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:calo_deposit -c 1 -o /tmp/ncu/dep6 python bench.py --workload c5_full --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py /tmp/ncu/dep6.ncu-rep > gpurun_out/r2_ncu_calo_deposit.txt 2>&1
cat gpurun_out/r2_ncu_calo_deposit.txt
rm -f gpurun_out/sanitizer.txt
bash tools/sanitize.sh
