#!/usr/bin/env python3
"""A/B timing of libprng_b200.so variants (tools/build_variants.sh).

tools/ab_lib.py WORKLOAD LOG2N ROUNDS tag1 tag2 ...  -- each variant runs in
its own process (PRNG_B200_LIB=build/var_<tag>/...), rounds interleave the
variants; prints per-variant median kernel ms / Gs/s and an output hash
(identical hashes = identical outputs, incl. a shifted-lane request).
"""
import hashlib
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

CHILD = r'''
import hashlib, json, sys, statistics
sys.path.insert(0, %r); sys.path.insert(0, %r)
import torch
import paper_2109_01329_b200 as P
from ncu_target import W
name, n = %r, 1 << %d
eng, mk, dt = W[name]
st = P.seed_engine(P.EngineKind.PHILOX4X32X10 if eng == "philox" else P.EngineKind.MRG32K3A, 777)
spec = mk()
h = hashlib.sha256()
for skip, m in ((0, 1 << 22), (1, (1 << 22) + 7), (3, 1000003)):
    _, o = P.generate(spec, P.skip_ahead(st, skip) if skip else st, m)
    h.update(o.cpu().numpy().tobytes())
out = torch.empty(n, dtype=dt, device="cuda")
for _ in range(5):
    P.generate(spec, st, n, out=out)
torch.cuda.synchronize()
ts = []
for _ in range(30):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); P.generate(spec, st, n, out=out); b.record(); b.synchronize()
    ts.append(a.elapsed_time(b))
print(json.dumps({"ms": statistics.median(ts), "min": min(ts), "hash": h.hexdigest()[:16]}))
'''


def main():
    wl, lg, rounds = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    tags = sys.argv[4:]
    res = {t: [] for t in tags}
    hashes = {}
    for r in range(rounds):
        for t in tags:
            env = dict(os.environ, PRNG_B200_LIB=str(ROOT / "build" / f"var_{t}" / "libprng_b200.so"))
            if t == "main":
                env.pop("PRNG_B200_LIB")
            code = CHILD % (str(ROOT), str(ROOT / "tools"), wl, lg)
            out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
            if out.returncode:
                print(t, "FAILED", out.stderr[-800:])
                continue
            d = json.loads(out.stdout.strip().splitlines()[-1])
            res[t].append(d["ms"])
            hashes[t] = d["hash"]
    n = 1 << lg
    for t in tags:
        if res[t]:
            ms = statistics.median(res[t])
            print(f"{wl} 2^{lg} {t:10s} median {ms:.4f} ms  best {min(res[t]):.4f}  {n / ms / 1e6:8.1f} Gs/s  hash {hashes[t]}")


if __name__ == "__main__":
    main()
