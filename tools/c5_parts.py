#!/usr/bin/env python3
"""C5 critical-path parts on the GPU box: the D2H of the run's packed
deposits alone (same bytes, same 5-chunk split, pinned destination), the
whole simulate_events, and a cProfile of its host side (tottime)."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2109_01329_b200 as P
from paper_2109_01329_b200 import calosim as C

nev, regions, ncells = 10000, 24, 190_000
geom = [np.arange(r, ncells, regions, dtype=np.int64) for r in range(regions)]
edges = np.linspace(0.001, 0.101, 9)
weights = np.asarray([0.05, 0.10, 0.20, 0.25, 0.20, 0.10, 0.07, 0.03])
det = C.Detector(geom, {"electron": C.Parameterization("electron", 4000, 6500, edges, weights)})
events = C.synth_single_electron_events(nev, 777)
st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
for _ in range(3):
    final, res = C.simulate_events(events, det, st, dicts=False)
torch.cuda.synchronize()
ts = []
for _ in range(8):
    t0 = time.perf_counter()
    final, res = C.simulate_events(events, det, st, dicts=False)
    torch.cuda.synchronize()
    ts.append(1e3 * (time.perf_counter() - t0))
print("simulate_events ms:", " ".join(f"{t:.2f}" for t in ts))
ndep = len(res["cells"])
dc = torch.empty(ndep, dtype=torch.int32, device="cuda")
de = torch.empty(ndep, dtype=torch.float64, device="cuda")
hc = torch.empty(ndep, dtype=torch.int32, pin_memory=True)
he = torch.empty(ndep, dtype=torch.float64, pin_memory=True)
cs = torch.cuda.Stream()
for split in (1, 5):
    bounds = np.linspace(0, ndep, split + 1).astype(np.int64)
    tt = []
    for _ in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(cs):
            for a, b in zip(bounds[:-1], bounds[1:]):
                hc[a:b].copy_(dc[a:b], non_blocking=True)
                he[a:b].copy_(de[a:b], non_blocking=True)
        cs.synchronize()
        tt.append(1e3 * (time.perf_counter() - t0))
    print(f"D2H of {ndep} deposits ({ndep * 12 / 1e6:.0f} MB) in {split} chunk(s) ms:", " ".join(f"{t:.2f}" for t in tt))
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    C.simulate_events(events, det, st, dicts=False)
    torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
