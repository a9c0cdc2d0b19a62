# Round 2 pass 40: SASS-level samples of the deposit kernel (report from pass 27 if the box kept /tmp, else recapture).
mkdir -p gpurun_out /tmp/ncu
[ -f /tmp/ncu/dep6.ncu-rep ] || timeout 600 ncu --set full --clock-control none --import-source on -k regex:calo_deposit -c 1 -o /tmp/ncu/dep6 python bench.py --workload c5_full --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ncu -i /tmp/ncu/dep6.ncu-rep --page source --csv --print-source sass 2>&1 | gzip -c > gpurun_out/r2_40_dep_sass.csv.gz
ls -la gpurun_out/
