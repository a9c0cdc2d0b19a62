# Round 2 pass 22: source-level profile of the deposit kernel.
mkdir -p gpurun_out /tmp/ncu
rm -f /tmp/ncu/dep*.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:calo_deposit -c 1 -o /tmp/ncu/dep2 python bench.py --workload c5_full --steps 1 --warmup 1 --no-cpu > gpurun_out/r2_22_ncu.log 2>&1
tail -5 gpurun_out/r2_22_ncu.log
python tools/ncu_summary.py /tmp/ncu/dep2.ncu-rep > gpurun_out/r2_22_dep_summary.txt 2>&1
ncu -i /tmp/ncu/dep2.ncu-rep --page source --csv --print-source sass > /tmp/ncu/dep_sass.csv 2>&1
ncu -i /tmp/ncu/dep2.ncu-rep --page source --csv --print-source cuda > /tmp/ncu/dep_cuda.csv 2>&1
ls -la /tmp/ncu/
gzip -c /tmp/ncu/dep_sass.csv > gpurun_out/r2_22_dep_sass.csv.gz
gzip -c /tmp/ncu/dep_cuda.csv > gpurun_out/r2_22_dep_cuda.csv.gz
cat gpurun_out/r2_22_dep_summary.txt
