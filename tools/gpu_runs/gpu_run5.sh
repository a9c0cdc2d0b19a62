mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r5_bench.json 2> gpurun_out/r5_bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r5_bench_ref.json 2> gpurun_out/r5_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5_launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/r5_bench_ncu.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:philox_kernel -s 3 -c 1 -o gpurun_out/r5_c4_full python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/r5_ncu_full.log 2>&1
cat gpurun_out/r5_bench.json gpurun_out/r5_bench_ref.json; tail -3 gpurun_out/r5_bench.err
