#!/usr/bin/env python3
"""Fit and exhaustively verify the fp32 polynomials of the fast Box-Muller path.

HISTORICAL: these were the polynomials of the first fast fp32 route; the
current route uses the SFU log/sqrt and a shared-memory sincos table
(csrc/common.cuh).  Kept as the record of the
exhaustive polynomial fits.

Emulates the device arithmetic in numpy float32 (FFMA as float64 fma then
one rounding to float32) over ALL 2^24 possible 24-bit inputs and reports the
error against float64 libm.  Prints C constants for common.cuh.
"""
import numpy as np

f32 = np.float32


def fma(a, b, c):
    return (a.astype(np.float64) * b.astype(np.float64) + c.astype(np.float64)).astype(np.float32)


def fit(fn, lo, hi, deg, weight=None):
    # least squares on Chebyshev nodes (close to minimax), float64
    k = np.arange(4000)
    x = (lo + hi) / 2 + (hi - lo) / 2 * np.cos(np.pi * (k + 0.5) / 4000)
    y = fn(x)
    w = np.ones_like(x) if weight is None else weight(x)
    V = np.vander(x, deg + 1, increasing=True)
    c, *_ = np.linalg.lstsq(V * w[:, None], y * w, rcond=None)
    return c


# --- ln(1+g) = g + g^2 * Q(g), g in [sqrt(.5)-1, sqrt(2)-1]
glo, ghi = np.sqrt(0.5) - 1, np.sqrt(2) - 1
Q = lambda g: np.where(np.abs(g) < 1e-8, -0.5 + g / 3, (np.log1p(g) - g) / np.where(g == 0, 1, g * g))
for deg in (6, 7, 8):
    cq = fit(Q, glo, ghi, deg)
    cq32 = cq.astype(np.float32)
    g = np.linspace(glo, ghi, 200001).astype(np.float32)
    q = np.full_like(g, cq32[-1])
    for c in cq32[-2::-1]:
        q = fma(q, g, np.full_like(g, c))
    l = fma(g * g, q, g)
    ref = np.log1p(g.astype(np.float64))
    err = np.abs(l.astype(np.float64) - ref) / np.maximum(np.abs(ref), 1e-30)
    print(f"ln poly deg {deg}: max rel err {err.max():.3e} ({err.max()/2**-24:.2f} ulp-ish)")
LN_DEG = 7
CQ = fit(Q, glo, ghi, LN_DEG).astype(np.float32)

# --- sin(pi/4 t) = t * S(t^2), cos(pi/4 t) = C(t^2), t in [-1, 1]
S = lambda u: np.where(u == 0, np.pi / 4, np.sin(np.pi / 4 * np.sqrt(u)) / np.sqrt(np.maximum(u, 1e-300)))
C = lambda u: np.cos(np.pi / 4 * np.sqrt(u))
CS = fit(S, 0, 1, 4).astype(np.float32)
CC = fit(C, 0, 1, 4).astype(np.float32)


def dev_log_m2(m):
    """-2 ln(m * 2^-24) for integer m in [1, 2^24], device emulation."""
    x = m.astype(np.float32)  # exact (m <= 2^24)
    ib = x.view(np.int32)
    e = (ib - np.int32(0x3F3504F3)) >> 23
    fb = ib - (e << 23)
    f = fb.view(np.float32)
    g = (f - f32(1.0)).astype(np.float32)
    q = np.full_like(g, CQ[-1])
    for c in CQ[-2::-1]:
        q = fma(q, g, np.full_like(g, c))
    l = fma((g * g).astype(np.float32), q, g)  # ln f
    et = (e - 24).astype(np.float32)
    ln2 = f32(0.6931471805599453)
    lnx = fma(et, np.full_like(et, ln2), l)
    return (lnx * f32(-2.0)).astype(np.float32)


def dev_sincos(k):
    kk = k + (1 << 21)
    q = (kk >> 22) & 3
    r = (kk & 0x3FFFFF).astype(np.int64) - (1 << 21)
    t = (r.astype(np.float32) * f32(2.0 ** -21)).astype(np.float32)
    t2 = (t * t).astype(np.float32)
    s = np.full_like(t2, CS[-1])
    for c in CS[-2::-1]:
        s = fma(s, t2, np.full_like(t2, c))
    s = (s * t).astype(np.float32)
    c_ = np.full_like(t2, CC[-1])
    for c in CC[-2::-1]:
        c_ = fma(c_, t2, np.full_like(t2, c))
    swap = (q & 1) == 1
    cs = np.where(swap, s, c_)
    sn = np.where(swap, c_, s)
    negc = ((q + 1) >> 1) & 1
    negs = q >> 1
    cs = np.where(negc == 1, -cs, cs)
    sn = np.where(negs == 1, -sn, sn)
    return sn.astype(np.float32), cs.astype(np.float32)


def main():
    m = np.arange(1, (1 << 24) + 1, dtype=np.int64)
    s = dev_log_m2(m)
    ref = -2.0 * np.log(m.astype(np.float64) / 2**24)
    rel = np.abs(s.astype(np.float64) - ref) / np.maximum(ref, 1e-300)
    rel[ref == 0] = np.abs(s[ref == 0])
    print(f"-2 ln x: max rel err {rel.max():.3e} = {rel.max()/2**-24:.2f} x 2^-24")
    # r = sqrt(s) via rsqrt (MUFU ~ 2^-22.9 rel): r rel err <= rel/2 + 2^-22.9
    k = np.arange(1 << 24, dtype=np.int64)
    sn, cs = dev_sincos(k)
    ang = 2 * np.pi * k / 2**24
    es = np.abs(sn.astype(np.float64) - np.sin(ang)).max()
    ec = np.abs(cs.astype(np.float64) - np.cos(ang)).max()
    print(f"sin abs err {es:.3e} ({es/2**-24:.2f} x 2^-24), cos abs err {ec:.3e} ({ec/2**-24:.2f} x 2^-24)")
    fmt = lambda a: ", ".join(f"{float(v):.9e}f" for v in a)
    print(f"LN_Q[{len(CQ)}] = {{{fmt(CQ)}}};")
    print(f"SIN_S[{len(CS)}] = {{{fmt(CS)}}};")
    print(f"COS_C[{len(CC)}] = {{{fmt(CC)}}};")


if __name__ == "__main__":
    main()
