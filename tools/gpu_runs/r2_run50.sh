# Round 2 pass 50: SASS-level samples of the normalisation kernel.
mkdir -p gpurun_out /tmp/ncu
rm -f /tmp/ncu/norm.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:calo_normalize -c 1 -o /tmp/ncu/norm python bench.py --workload c5_full --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ncu -i /tmp/ncu/norm.ncu-rep --page source --csv --print-source sass 2>&1 | gzip -c > gpurun_out/r2_50_norm_sass.csv.gz
python tools/ncu_summary.py /tmp/ncu/norm.ncu-rep
