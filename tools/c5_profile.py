#!/usr/bin/env python3
"""cProfile of calosim.simulate_events (C5 full, 10^4 single-electron
events, dicts=False) on the GPU box: where the host time goes."""
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
for _ in range(2):
    C.simulate_events(events, det, st, dicts=False)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    C.simulate_events(events, det, st, dicts=False)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print("wall ms per run:", [round(t * 1e3, 2) for t in ts])
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    C.simulate_events(events, det, st, dicts=False)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
