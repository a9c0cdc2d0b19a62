import sys, time, gc
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2109_01329_b200 as P
from paper_2109_01329_b200 import calosim as C
nev, regions, ncells = 10000, 24, 190_000
geom = [np.arange(r, ncells, regions, dtype=np.int64) for r in range(regions)]
edges = np.linspace(0.001, 0.101, 9)
weights = np.asarray([0.05, 0.10, 0.20, 0.25, 0.20, 0.10, 0.07, 0.03])
det = C.Detector(geom, {"electron": C.Parameterization("electron", 4000, 6500, edges, weights)})
events = C.synth_single_electron_events(nev, 777)
st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
for mode in ("hold", "drop", "hold_gcoff"):
    if mode == "hold_gcoff": gc.disable()
    res = None
    ts = []
    for i in range(18):
        t0 = time.perf_counter()
        if mode == "drop":
            res = None
        final, res = C.simulate_events(events, det, st, dicts=False)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(mode, " ".join(f"{t:.1f}" for t in ts))
    gc.enable()
