mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 | grep -E "^\{" | head -2
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1
