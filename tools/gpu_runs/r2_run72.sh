# Round 2 pass 72: SASS-level samples of the exact fp32 gaussian kernel.
mkdir -p gpurun_out /tmp/ncu
rm -f /tmp/ncu/ex.ncu-rep
timeout 600 ncu --set full --clock-control none --import-source on -k regex:philox_kernel -c 1 -s 1 -o /tmp/ncu/ex python tools/ncu_target.py gauss_f32_exact 28 3 > /dev/null 2>&1
ncu -i /tmp/ncu/ex.ncu-rep --page source --csv --print-source sass 2>&1 | gzip -c > gpurun_out/r2_72_exact_sass.csv.gz
python tools/ncu_summary.py /tmp/ncu/ex.ncu-rep | head -20
