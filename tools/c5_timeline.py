#!/usr/bin/env python3
"""Host-side timeline of one calosim.simulate_events call (C5 full, 10^4
single-electron events): wraps the module's helpers with perf_counter
stamps and prints when each starts / ends relative to the call, to show
what sits on the critical path before the first D2H and after the last."""
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
log = []
T0 = [0.0]


def wrap(mod, name):
    f = getattr(mod, name)

    def g(*a, **k):
        t = time.perf_counter()
        r = f(*a, **k)
        log.append((name, (t - T0[0]) * 1e3, (time.perf_counter() - T0[0]) * 1e3))
        return r
    setattr(mod, name, g)


for n in ("_particle_columns", "_plan_fixed_from_draws", "_particle_table_arrays",
          "generate_segments"):
    wrap(C, n)
orig_sync = torch.cuda.Event.synchronize


def ev_sync(self):
    t = time.perf_counter()
    orig_sync(self)
    log.append(("Event.synchronize", (t - T0[0]) * 1e3, (time.perf_counter() - T0[0]) * 1e3))


torch.cuda.Event.synchronize = ev_sync
for _ in range(3):
    C.simulate_events(events, det, st, dicts=False)
torch.cuda.synchronize()
for it in range(3):
    log.clear()
    T0[0] = time.perf_counter()
    C.simulate_events(events, det, st, dicts=False)
    torch.cuda.synchronize()
    tot = (time.perf_counter() - T0[0]) * 1e3
    print(f"--- call {it}: {tot:.2f} ms")
    for name, a, b in log:
        print(f"  {a:8.2f} -> {b:8.2f} ms  ({b - a:6.2f})  {name}")
