# Round-1 refresh: tests, every bench workload, launch list + ncu full captures.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu --durations=8 2>&1 | tail -20 > gpurun_out/r11_pytest.txt
timeout 600 python bench.py > gpurun_out/r11_c4.json 2> gpurun_out/r11_c4.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r11_reference.json 2>/dev/null
timeout 600 python bench.py --workload c5 --steps 10 > gpurun_out/r11_c5.json 2> gpurun_out/r11_c5.err
timeout 600 python bench.py --workload c5_full --steps 5 --warmup 3 > gpurun_out/r11_c5_full.json 2> gpurun_out/r11_c5_full.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --sweep > gpurun_out/r11_sweep.json 2> gpurun_out/r11_sweep.err
for w in c2 c3_gauss c3_logn c4_bits c1; do timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r11_$w.json 2>gpurun_out/r11_$w.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r11_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r11_launches_c5_full.csv python bench.py --workload c5_full --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
for w in unit_f32 mrg_bits mrg_f64 gauss_f32; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:"mrg|philox" -c 1 -s 1 -o gpurun_out/r11_$w python tools/ncu_target.py $w 28 3 > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"philox" -c 1 -s 1 -o gpurun_out/r11_c4_2p32 python tools/ncu_target.py unit_f32 32 2 > /dev/null 2>&1
cat gpurun_out/r11_pytest.txt | tail -12
for f in c4 reference c5 c5_full c2 c3_gauss c3_logn c4_bits c1; do echo "$f: $(head -c 400 gpurun_out/r11_$f.json)"; done
