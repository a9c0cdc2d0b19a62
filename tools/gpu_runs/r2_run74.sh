# Round 2 pass 74: ncu summaries of the final C5 kernels (deposit, normalisation, hits, segments).
mkdir -p gpurun_out /tmp/ncu
rm -f /tmp/ncu/c5k.ncu-rep
timeout 600 ncu --set full --clock-control none -k regex:"calo_|philox_segments" -c 8 -o /tmp/ncu/c5k python bench.py --workload c5_full --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py /tmp/ncu/c5k.ncu-rep > gpurun_out/r2_ncu_c5_kernels.txt 2>&1
grep -E "^kernel|gpu__time|issue_active|dram__bytes_write|stalls" gpurun_out/r2_ncu_c5_kernels.txt | head -40
