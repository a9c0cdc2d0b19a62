# Round-1 refresh part A: tests, every bench workload, launch lists.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3 > gpurun_out/r13_pytest.txt
timeout 600 python bench.py > gpurun_out/r13_c4.json 2> gpurun_out/r13_c4.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r13_reference.json 2>/dev/null
timeout 600 python bench.py --workload c5 --steps 10 > gpurun_out/r13_c5.json 2> gpurun_out/r13_c5.err
timeout 600 python bench.py --workload c5_full --steps 5 --warmup 3 > gpurun_out/r13_c5_full.json 2> gpurun_out/r13_c5_full.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --sweep > gpurun_out/r13_sweep.json 2> gpurun_out/r13_sweep.err
for w in c2 c3_gauss c3_logn c4_bits c1; do timeout 300 python bench.py --workload $w --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r13_$w.json 2>gpurun_out/r13_$w.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r13_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r13_launches_c5_full.csv python bench.py --workload c5_full --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
du -sh gpurun_out
