#!/usr/bin/env python3
"""Quick device-side throughput probe of every kernel family (not the bench).

Prints one line per (workload, n): kernel ms (CUDA events, median of reps),
Gsamples/s and GB/s of algorithmic writes; plus torch's own fill_ of the same
buffer as a write-only bandwidth reference.
"""
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
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ph = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
    mr = P.seed_engine(P.EngineKind.MRG32K3A, 777)
    cases = [
        ("fill_f32 (torch)", None, None, torch.float32, 1 << 32),
        ("philox unit f32", ph, P.Uniform(0.0, 1.0), torch.float32, 1 << 32),
        ("philox unit f32 lane1", P.skip_ahead(ph, 1), P.Uniform(0.0, 1.0), torch.float32, 1 << 32),
        ("philox uniform f32 [-3,5)", ph, P.Uniform(-3.0, 5.0), torch.float32, 1 << 32),
        ("philox bits", ph, P.UniformBits(), torch.uint32, 1 << 32),
        ("philox unit f64", ph, P.Uniform(0.0, 1.0, "fp64"), torch.float64, 1 << 31),
        ("philox gauss f32 fast", ph, P.Gaussian(0.0, 1.0), torch.float32, 1 << 30),
        ("philox gauss f32 acc", ph, P.Gaussian(0.0, 1.0, method="accurate"), torch.float32, 1 << 30),
        ("philox gauss f64", ph, P.Gaussian(0.0, 1.0, "fp64"), torch.float64, 1 << 29),
        ("philox gauss f32 exact", ph, P.Gaussian(0.0, 1.0, method="exact"), torch.float32, 1 << 30),
        ("philox gauss f64 exact", ph, P.Gaussian(0.0, 1.0, "fp64", "exact"), torch.float64, 1 << 29),
        ("philox logn f32 fast", ph, P.Lognormal(), torch.float32, 1 << 30),
        ("mrg bits", mr, P.UniformBits(), torch.uint32, 1 << 28),
        ("mrg uniform f64 [-1,1)", mr, P.Uniform(-1.0, 1.0, "fp64"), torch.float64, 1 << 28),
        ("mrg uniform f32", mr, P.Uniform(0.0, 1.0), torch.float32, 1 << 28),
        ("mrg gauss f32", mr, P.Gaussian(0.0, 1.0), torch.float32, 1 << 28),
    ]
    for name, st, spec, dt, n in cases:
        out = torch.empty(n, dtype=dt, device="cuda")
        if st is None:
            fn = lambda: out.fill_(1.0)
        else:
            fn = lambda: P.generate(spec, st, n, out=out)
        ms = timeit(fn)
        gb = n * out.element_size() / ms / 1e6
        print(f"{name:28s} n=2^{n.bit_length()-1:<3d} {ms:9.3f} ms  {n/ms/1e6:9.1f} Gs/s  {gb:8.1f} GB/s", flush=True)
        del out
        torch.cuda.empty_cache()
    # small sizes: launch-bound regime
    for k in (10, 14, 18, 20, 22, 24, 26, 28, 30):
        n = 1 << k
        out = torch.empty(n, dtype=torch.float32, device="cuda")
        ms = timeit(lambda: P.generate(P.Uniform(0.0, 1.0), ph, n, out=out), reps=50)
        print(f"sweep unit f32 n=2^{k:<3d} {ms*1e3:9.1f} us  {n/ms/1e6:9.1f} Gs/s", flush=True)


if __name__ == "__main__":
    main()
