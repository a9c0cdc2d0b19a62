"""bench.py host logic on CPU: the per-rank slice check accepts the
single-stream oracle's own slice for every workload and rejects a corrupted
one (no GPU: `out` is a CPU tensor built from the oracle)."""

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

import bench  # noqa: E402
import paper_2109_01329_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def _slice(workload, n, rank):
    engine, dist, prec, _, _ = bench.WORKLOADS[workload]
    g = rank * n
    st = (O.seed_philox(777), g) if engine == "philox" else O.mrg_skip(*O.seed_mrg(777), g)
    a, b = (-1.0, 1.0) if (dist == "uniform" and prec == "fp64") else (0.0, 1.0)
    return O.generate(engine, st, dist, n, prec, a, b)


@pytest.mark.parametrize("workload", ["c1", "c4", "c4_bits", "c2", "c3_gauss", "c3_logn", "c3_gauss_precise",
                                      "c3_logn_precise", "c3_gauss_exact"])
@pytest.mark.parametrize("rank", [0, 3])
def test_slice_check_accepts_oracle_slices(workload, rank):
    n = 1 << 14
    engine, dist, prec, _, _ = bench.WORKLOADS[workload]
    spec = bench.make_spec(P, dist, prec, bench.WORKLOAD_METHOD.get(workload, "fast"))
    want = _slice(workload, n, rank)
    ok, worst = bench.slice_check(P, torch, workload, spec, torch.from_numpy(want.copy()), n, rank)
    assert ok and worst <= 1.0
    bad = want.copy()
    bad[-1] = bad[-1] + (1 if bad.dtype == np.uint32 else bad[-1] * 1e-3 + 1e-3)
    ok, _ = bench.slice_check(P, torch, workload, spec, torch.from_numpy(bad), n, rank)
    assert not ok
    if rank:  # another rank's slice is not this rank's
        other = _slice(workload, n, 0)
        assert not bench.slice_check(P, torch, workload, spec, torch.from_numpy(other), n, rank)[0]
