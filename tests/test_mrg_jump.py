"""CPU check of the MRG32k3a segment jump used by mrg_kernel (mrg32k3a.cuh
mrg_jump, api.cu split_jump): x -> B x mod m with B = A^(31*seg) split into
16-bit halves and evaluated in fp64 must equal the big-integer product for
every symmetric-residue state, and must land back in [-m/2 - 1, m/2 + 1].

The fp64 operations are replayed exactly rounded (products and FMAs through
fractions), the way the device evaluates __dmul_rn / __fma_rn.
"""
from fractions import Fraction
import random

import pytest

M1 = 2**32 - 209
M2 = 2**32 - 22853
A1 = [[0, 1, 0], [0, 0, 1], [(M1 - 810728) % M1, 1403580, 0]]  # engine.py:165-174
A2 = [[0, 1, 0], [0, 0, 1], [(M2 - 1370589) % M2, 0, 527612]]
MAGIC = 6755399441055744.0  # 1.5 * 2^52


def matmul(a, b, m):
    return [[sum(a[i][k] * b[k][j] for k in range(3)) % m for j in range(3)] for i in range(3)]


def matpow(a, k, m):
    r = [[1, 0, 0], [0, 1, 0], [0, 0, 1]]
    while k:
        if k & 1:
            r = matmul(r, a, m)
        a = matmul(a, a, m)
        k >>= 1
    return r


def fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def reduce_(p, m):  # mrg_reduce (common.cuh)
    k = fma(p, 1.0 / m, MAGIC) - MAGIC
    return fma(-k, float(m), p)


def sym(x, m):
    return x - m if x > m // 2 else x


def split(b, m):  # split_jump (api.cu)
    hi, lo = [], []
    for row in b:
        for v in row:
            v = sym(v, m)
            h = (v + 32768) // 65536 if v >= 0 else -((-v + 32767) // 65536)
            hi.append(float(h))
            lo.append(float(v - h * 65536))
    return hi, lo


@pytest.mark.parametrize("seg", [64, 128, 2368])
@pytest.mark.parametrize("comp", [1, 2])
def test_split_jump_is_exact(seg, comp):
    a, m = (A1, M1) if comp == 1 else (A2, M2)
    b = matpow(a, 31 * seg, m)
    hi, lo = split(b, m)
    assert max(abs(v) for v in hi + lo) <= 32768
    rng = random.Random(seg * 10 + comp)
    cases = [[m // 2, m // 2 + 1, m - 1], [0, 1, m - 1], [m // 2 + 1] * 3]
    cases += [[rng.randrange(m) for _ in range(3)] for _ in range(400)]
    for x in cases:
        xs = [float(sym(v, m)) for v in x]
        want = [sum(b[i][k] * x[k] for k in range(3)) % m for i in range(3)]
        got = []
        for i in range(3):
            l_ = fma(lo[3 * i + 2], xs[2], fma(lo[3 * i + 1], xs[1], lo[3 * i] * xs[0]))
            h_ = fma(hi[3 * i + 2], xs[2], fma(hi[3 * i + 1], xs[1], hi[3 * i] * xs[0]))
            got.append(reduce_(fma(reduce_(h_, m), 65536.0, l_), m))
        assert all(abs(v) <= m / 2 + 1 for v in got)
        assert [int(v) % m for v in got] == want
