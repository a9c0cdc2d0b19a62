#!/usr/bin/env python3
"""Host-side cost per generate() call for tiny requests (launch-bound regime)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2109_01329_b200 as P
from paper_2109_01329_b200 import _lib


def per_call(fn, n=5000):
    for _ in range(100):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e6


st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
out = torch.empty(1024, device="cuda")
spec = P.Uniform(0.0, 1.0)
print(f"generate(spec, state, 1024, out)          {per_call(lambda: P.generate(spec, st, 1024, out=out)):7.2f} us")
print(f"generate(spec, state, 1024) [alloc]       {per_call(lambda: P.generate(spec, st, 1024)):7.2f} us")
k0, k1, ctr, lane = P.engine.philox_args(st)
s = torch.cuda.current_stream().cuda_stream
ptr = out.data_ptr()
f = _lib.lib.prng_philox4x32x10_uniform_f32
print(f"raw C-ABI call                            {per_call(lambda: f(k0, k1, ctr, lane, 1024, 0.0, 1.0, ptr, s)):7.2f} us")
if hasattr(P, "Philox4x32x10"):
    eng = P.Philox4x32x10(777)
    print(f"engine object generate                    {per_call(lambda: P.generate(spec, eng, 1024, out=out)):7.2f} us")
