# Round 2 pass 53: N=2 functional dry run at HEAD (two torchrun ranks sharing the one B200 over gloo) and
# bench --gpus 2 self-launch path.
mkdir -p gpurun_out
PRNG_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2_53_g2_share.json 2> gpurun_out/r2_53_g2_share.err
echo "rc=$?"; tail -c 1500 gpurun_out/r2_53_g2_share.json; tail -5 gpurun_out/r2_53_g2_share.err
PRNG_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/r2_53_g2_ref.json 2> gpurun_out/r2_53_g2_ref.err
echo "ref rc=$?"; tail -c 400 gpurun_out/r2_53_g2_ref.json
