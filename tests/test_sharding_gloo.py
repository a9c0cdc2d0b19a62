"""Multi-rank sharding logic on CPU: world_size-2 gloo processes.

Each rank computes its shard (bench.py's weak and strong layouts), its start
state via skip_ahead, and the oracle's words for that shard; rank 0 gathers
the slices and checks that their concatenation equals the single-stream
oracle -- the same property the GPU test checks with device slices.  The
GPU kernels are not called here (no device); the sharding arithmetic and
state placement are the host logic under test.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_slice(spec_kind, state, count):
    from oracle import oracle as O
    import paper_2109_01329_b200 as P

    if isinstance(state, P.PhiloxState):
        st = ("philox", (state.key, P.stream_position(state)))
    else:
        st = ("mrg", (state.s1, state.s2))
    if spec_kind == "uniform":
        return O.generate(st[0], st[1], "uniform", count, "fp32", 0.0, 1.0)
    return O.generate(st[0], st[1], "gaussian", count, "fp64", 0.0, 1.0)


def _worker(rank, world, port, results):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2109_01329_b200 as P
    from paper_2109_01329_b200.sharding import shard_state, strong_shard, weak_shard

    ok = True
    for engine in (P.EngineKind.PHILOX4X32X10, P.EngineKind.MRG32K3A):
        base = P.seed_engine(engine, 777)
        for kind, spec in (("uniform", P.Uniform(0.0, 1.0)), ("gaussian", P.Gaussian(0.0, 1.0, "fp64"))):
            for shard in (strong_shard(10_001, rank, world), weak_shard(4096, rank, world)):
                st = shard_state(spec, base, shard)
                part = torch.from_numpy(_oracle_slice(kind, st, shard.count).astype(np.float64))
                sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
                dist.all_gather(sizes, torch.tensor([part.numel()]))
                mx = int(max(s.item() for s in sizes))
                padded = torch.zeros(mx, dtype=torch.float64)
                padded[: part.numel()] = part
                gathered = [torch.zeros(mx, dtype=torch.float64) for _ in range(world)]
                dist.all_gather(gathered, padded)
                if rank == 0:
                    full = torch.cat([g[: int(s.item())] for g, s in zip(gathered, sizes)]).numpy()
                    total = sum(int(s.item()) for s in sizes)
                    want = _oracle_slice(kind, base, total).astype(np.float64)
                    ok &= np.array_equal(full, want)
    dist.destroy_process_group()
    results[rank] = ok


@pytest.mark.timeout(300)
def test_world2_shards_concatenate_to_single_stream():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, results)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0
    assert results[0] is True


def test_strong_shard_partitions_exactly():
    from paper_2109_01329_b200.sharding import strong_shard

    for n in (0, 1, 7, 4096, 10_001, (1 << 32) + 3):
        for world in (1, 2, 3, 8):
            shards = [strong_shard(n, r, world) for r in range(world)]
            assert shards[0].start == 0
            for a, b in zip(shards, shards[1:]):
                assert a.start + a.count == b.start
                assert b.start % 4 == 0
            assert shards[-1].start + shards[-1].count == n
