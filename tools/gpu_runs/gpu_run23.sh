# ncu --set full DRAM traffic for the non-headline bench kernels (c4_bits 2^32, c2 2^28, c3 2^30) + torchrun N=1 path.
mkdir -p gpurun_out
for spec in "c4_bits bits 32" "c2 mrg_f64 28" "c3_gauss gauss_f32 30" "c3_logn logn_f32 30"; do
  set -- $spec
  timeout 400 ncu --set full --clock-control none -k regex:"mrg|philox" -c 1 -s 1 -o gpurun_out/r23_$1 python tools/ncu_target.py $2 $3 2 > gpurun_out/r23_ncu_$1.log 2>&1
  ncu -i gpurun_out/r23_$1.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active > gpurun_out/r23_$1_raw.csv 2>&1
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu > gpurun_out/r23_torchrun1.json 2> gpurun_out/r23_torchrun1.err
for lg in 30 31 32; do timeout 200 python tools/ab_lib.py unit_f32 $lg 3 main >> gpurun_out/r23_sizes.txt 2>&1; done
cat gpurun_out/r23_*_raw.csv gpurun_out/r23_torchrun1.json gpurun_out/r23_sizes.txt; tail -3 gpurun_out/r23_torchrun1.err
