#!/usr/bin/env python3
"""MRG32k3a kernel throughput probe (device time, CUDA events, median of 20)."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2109_01329_b200 as P


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


st = P.seed_engine(P.EngineKind.MRG32K3A, 777)
n = 1 << 28
for name, spec, dt in (("mrg bits", P.UniformBits(), torch.uint32),
                       ("mrg uniform f64 [-1,1)", P.Uniform(-1.0, 1.0, "fp64"), torch.float64),
                       ("mrg uniform f32", P.Uniform(0.0, 1.0), torch.float32),
                       ("mrg gauss f32", P.Gaussian(0.0, 1.0), torch.float32)):
    out = torch.empty(n, dtype=dt, device="cuda")
    ms = timeit(lambda: P.generate(spec, st, n, out=out))
    print(f"{name:24s} n=2^28 {ms:8.3f} ms {n / ms / 1e6:8.1f} Gs/s {n * out.element_size() / ms / 1e6:8.1f} GB/s")
