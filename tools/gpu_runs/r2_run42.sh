# Round 2 pass 42: SASS-level samples of the current deposit kernel.
mkdir -p gpurun_out /tmp/ncu
rm -f /tmp/ncu/dep8.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:calo_deposit -c 1 -o /tmp/ncu/dep8 python bench.py --workload c5_full --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ncu -i /tmp/ncu/dep8.ncu-rep --page source --csv --print-source sass 2>&1 | gzip -c > gpurun_out/r2_42_dep_sass.csv.gz
ls -la gpurun_out
