#!/usr/bin/env python3
"""What Python's cyclic GC walks during the C5 run: tracked objects by type
and the cost of a full collection, before and after simulate_events."""
import gc
import sys
import time
from collections import Counter
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2109_01329_b200 as P
from paper_2109_01329_b200 import calosim as C


def full():
    t = time.perf_counter()
    gc.collect()
    return (time.perf_counter() - t) * 1e3


print(f"after imports: {len(gc.get_objects())} tracked, full collection {full():.1f} ms")
nev, regions, ncells = 10000, 24, 190_000
geom = [np.arange(r, ncells, regions, dtype=np.int64) for r in range(regions)]
edges = np.linspace(0.001, 0.101, 9)
weights = np.asarray([0.05, 0.10, 0.20, 0.25, 0.20, 0.10, 0.07, 0.03])
det = C.Detector(geom, {"electron": C.Parameterization("electron", 4000, 6500, edges, weights)})
events = C.synth_single_electron_events(nev, 777)
st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
print(f"with events: {len(gc.get_objects())} tracked, full collection {full():.1f} ms")
final, res = C.simulate_events(events, det, st, dicts=False)
torch.cuda.synchronize()
print(f"with a result: {len(gc.get_objects())} tracked, full collection {full():.1f} ms")
print("top tracked types:", Counter(type(o).__name__ for o in gc.get_objects()).most_common(8))
for gen in range(3):
    t = time.perf_counter()
    gc.collect(gen)
    print(f"collect({gen}) {1e3 * (time.perf_counter() - t):.2f} ms")
print("thresholds", gc.get_threshold(), "counts", gc.get_count())
