# Dry run of the N>1 bench path: 2 ranks sharing the one GPU (gloo), ours and the reference arm.
mkdir -p gpurun_out
PRNG_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 5 --warmup 3 --n-per-gpu 268435456 --e2e-n 67108864 > gpurun_out/r63_n2.json 2> gpurun_out/r63_n2.err; echo "rc=$?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/r63_ref2.json 2> gpurun_out/r63_ref2.err; echo "rc=$?"
cat gpurun_out/r63_n2.json gpurun_out/r63_ref2.json; tail -5 gpurun_out/r63_n2.err
