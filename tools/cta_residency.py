#!/usr/bin/env python3
"""CTA residency of the persistent Philox kernels: per-CTA (SM id, start, end)
from a PRNG_TRACE_CTA build (tools/build_variants.sh trace -DPRNG_TRACE_CTA).
PRNG_B200_LIB=build/var_trace/libprng_b200.so python tools/cta_residency.py WORKLOAD LOG2N"""
import ctypes
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import numpy as np
import torch

import paper_2109_01329_b200 as P
from paper_2109_01329_b200 import _lib
from ncu_target import W

name, lg = sys.argv[1], int(sys.argv[2])
eng, mk, dt = W[name]
st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
out = torch.empty(1 << lg, dtype=dt, device="cuda")
spec = mk()
for _ in range(3):
    P.generate(spec, st, 1 << lg, out=out)
torch.cuda.synchronize()
f = _lib.lib.prng_diag_cta_trace
f.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros((8192, 3), dtype=np.uint64)
assert f(buf.ctypes.data, 8192) == 0
rows = buf[buf[:, 2] > 0]
sm, t0, t1 = rows[:, 0].astype(int), rows[:, 1].astype(np.int64), rows[:, 2].astype(np.int64)
base = t0.min()
t0, t1 = (t0 - base) / 1e3, (t1 - base) / 1e3  # us
dur = t1 - t0
per_sm = defaultdict(list)
for s, a, b in zip(sm, t0, t1):
    per_sm[s].append((a, b))
counts = np.array([len(v) for v in per_sm.values()])
# max concurrency per SM: sweep events
conc = []
for v in per_sm.values():
    ev = sorted([(a, 1) for a, _ in v] + [(b, -1) for _, b in v])
    c = m = 0
    for _, d in ev:
        c += d
        m = max(m, c)
    conc.append(m)
span = t1.max()
busy = sum(dur) / (len(per_sm) * span)
print(f"{name} 2^{lg}: {len(rows)} CTAs on {len(per_sm)} SMs; CTAs/SM min {counts.min()} max {counts.max()}; "
      f"max concurrent/SM min {min(conc)} max {max(conc)}; kernel span {span:.1f} us")
print(f"  CTA start: min {t0.min():.1f} median {np.median(t0):.1f} max {t0.max():.1f} us; "
      f"CTA duration: min {dur.min():.1f} median {np.median(dur):.1f} max {dur.max():.1f} us; "
      f"mean resident CTAs/SM {busy * counts.mean():.2f}")
late = t0 > 0.05 * span
print(f"  CTAs starting after 5% of the span: {late.sum()}")
