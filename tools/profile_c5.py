#!/usr/bin/env python3
"""Stage timing of calosim.simulate_events (host planning vs GPU kernels vs D2H)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import cProfile
import pstats

import numpy as np
import torch

import paper_2109_01329_b200 as P
from paper_2109_01329_b200 import calosim as C

nev, regions, ncells = int(sys.argv[1]) if len(sys.argv) > 1 else 10000, 24, 190_000
geom = [np.arange(r, ncells, regions, dtype=np.int64) for r in range(regions)]
edges = np.linspace(0.001, 0.101, 9)
weights = np.asarray([0.05, 0.10, 0.20, 0.25, 0.20, 0.10, 0.07, 0.03])
det = C.Detector(geom, {"electron": C.Parameterization("electron", 4000, 6500, edges, weights)})
t0 = time.perf_counter()
events = C.synth_single_electron_events(nev, 777)
print(f"synth events {1e3 * (time.perf_counter() - t0):.1f} ms")
st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
C.simulate_events(events[:50], det, st, dicts=False)
torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter()
    C.simulate_events(events, det, st, dicts=False)
    torch.cuda.synchronize()
    print(f"simulate_events {1e3 * (time.perf_counter() - t0):.1f} ms")
pr = cProfile.Profile()
pr.enable()
C.simulate_events(events, det, st, dicts=False)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
