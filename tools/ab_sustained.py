#!/usr/bin/env python3
"""Sustained (power-capped) A/B of libprng_b200.so variants: 250 back-to-back
launches per variant, median of the last 150 (after the board has settled
under sw_power_cap), with 2 s of idle between variants.
tools/ab_sustained.py WORKLOAD LOG2N ROUNDS tag1 tag2 ..."""
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import json, sys, statistics
sys.path.insert(0, %r); sys.path.insert(0, %r)
import torch
import paper_2109_01329_b200 as P
from ncu_target import W
name, n = %r, 1 << %d
eng, mk, dt = W[name]
st = P.seed_engine(P.EngineKind.PHILOX4X32X10 if eng == "philox" else P.EngineKind.MRG32K3A, 777)
spec = mk()
out = torch.empty(n, dtype=dt, device="cuda")
for _ in range(3):
    P.generate(spec, st, n, out=out)
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(250)]
for a, b in ev:
    a.record(); P.generate(spec, st, n, out=out); b.record()
torch.cuda.synchronize()
ms = [a.elapsed_time(b) for a, b in ev]
print(json.dumps({"first": statistics.median(ms[:20]), "settled": statistics.median(ms[100:])}))
'''


def main():
    wl, lg, rounds = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    tags = sys.argv[4:]
    res = {t: [] for t in tags}
    for _ in range(rounds):
        for t in tags:
            env = dict(os.environ, PRNG_B200_LIB=str(ROOT / "build" / f"var_{t}" / "libprng_b200.so"))
            if t == "main":
                env.pop("PRNG_B200_LIB")
            out = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), str(ROOT / "tools"), wl, lg)], env=env,
                                 capture_output=True, text=True)
            if out.returncode:
                print(t, "FAILED", out.stderr[-600:])
                continue
            res[t].append(json.loads(out.stdout.strip().splitlines()[-1]))
            time.sleep(2.0)
    n = 1 << lg
    for t in tags:
        if res[t]:
            f = statistics.median(r["first"] for r in res[t])
            s = statistics.median(r["settled"] for r in res[t])
            print(f"{wl} 2^{lg} {t:8s} first {f:.4f} ms ({n / f / 1e6:7.1f} Gs/s)  settled {s:.4f} ms ({n / s / 1e6:7.1f} Gs/s)")


if __name__ == "__main__":
    main()
