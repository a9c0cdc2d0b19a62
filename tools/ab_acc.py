#!/usr/bin/env python3
"""Accuracy of fast fp32 gaussian/lognormal variants (tools/build_variants.sh):
exhaustive 2^24 u1 / u2 sweep (as tests/test_gpu_parity.py
test_box_muller_exhaustive_24bit) plus a dense lognormal stream; prints the
max err/allowed ratio per variant (must be <= 1).
tools/ab_acc.py tag1 tag2 ..."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CHILD = r'''
import sys
sys.path.insert(0, %r); sys.path.insert(0, %r)
import numpy as np, torch
import paper_2109_01329_b200 as P
from oracle import oracle as O
from tolerances import gaussian_allowed, lognormal_allowed
k = np.arange(1 << 24, dtype=np.uint64)
other = ((k * 2654435761) & 0xFFFFFF).astype(np.uint32)
kk = k.astype(np.uint32)
worst = 0.0; maxerr = 0.0
for first, second in ((kk, other), (other, kk)):
    words = np.empty(2 << 24, dtype=np.uint32)
    words[0::2] = first << np.uint32(8)
    words[1::2] = second << np.uint32(8)
    want = O.gaussian_from_words(words, 0.0, 1.0, 2 << 24, "fp32")
    got = P.gaussian_from_words(torch.from_numpy(words).cuda(), 0.0, 1.0, 2 << 24, "fp32", "fast").cpu().numpy()
    err = np.abs(got.astype(np.float64) - want.astype(np.float64))
    al = gaussian_allowed(want, 0.0, 1.0, np.float32, True)
    worst = max(worst, float(np.max(err / al))); maxerr = max(maxerr, float(err.max()))
lw = 0.0
st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
for (m, s, d, sc) in ((0.0, 1.0, 0.0, 1.0), (1.5, 0.25, 2.0, 3.0), (-2.0, 2.0, 0.0, 0.5)):
    n = 1 << 24
    _, got = P.generate(P.Lognormal(m, s, d, sc), st, n)
    want = O.generate("philox", (O.seed_philox(777), 0), "lognormal", n, "fp32", m, s, displ=d, scale=sc)
    al = lognormal_allowed((want.astype(np.float64) - d) / sc, m, s, np.float32, True) * sc + \
        4 * np.spacing(np.abs(want)).astype(np.float64)
    err = np.abs(got.cpu().numpy().astype(np.float64) - want.astype(np.float64))
    lw = max(lw, float(np.max(err / al)))
print(f"gauss max err {maxerr:.3e} worst err/allowed {worst:.3f}; lognormal worst {lw:.3f}")
'''
for t in sys.argv[1:]:
    env = dict(os.environ, PRNG_B200_LIB=str(ROOT / "build" / f"var_{t}" / "libprng_b200.so"))
    if t == "main":
        env.pop("PRNG_B200_LIB")
    out = subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), str(ROOT / "tests"))], env=env,
                         capture_output=True, text=True)
    print(t, out.stdout.strip() if out.returncode == 0 else "FAILED " + out.stderr[-1500:])
