"""Drop-in CUDA implementation of the reference kernel plugin.

Same module surface as pkg/src/portarng/_kernels/__init__.py:24-27 --
``IMPL``, ``philox_fill``, ``mrg_fill``, ``box_muller`` with the reference's
argument meaning and return types (fresh C-contiguous numpy arrays,
_core.pyx:42-122) -- backed by libprng_b200.so's host-buffer entry points
(prng_kernels_*: generate on the GPU, copy back).  INTEGRATION.md shows the
three-line change that lets portarng select it with PORTARNG_KERNELS=cuda.
"""

from __future__ import annotations

import ctypes

import numpy as np

from .. import _lib

IMPL = "cuda"


def _u32(v, name):
    v = int(v)
    if not 0 <= v <= 0xFFFFFFFF:
        # Cython's int -> uint32_t conversion raises OverflowError
        raise OverflowError(f"{name}={v} does not fit uint32")
    return v


def philox_fill(k0, k1, b0, b1, b2, b3, offset, n):
    """n Philox stream words starting at word `offset` of block (b0..b3) (_core.pyx:42)."""
    args = [_u32(x, nm) for x, nm in zip((k0, k1, b0, b1, b2, b3, offset), ("k0", "k1", "b0", "b1", "b2", "b3", "offset"))]
    n = int(n)
    out = np.empty(n, dtype=np.uint32)  # ValueError for n < 0, as np.empty in the reference
    if n:
        _lib.check(_lib.lib.prng_kernels_philox_fill(*args, n, out.ctypes.data))
    return out


def mrg_fill(s10, s11, s12, s20, s21, s22, n):
    """n MRG32k3a words plus the advanced windows (_core.pyx:74)."""
    st = [_u32(x, "state") for x in (s10, s11, s12, s20, s21, s22)]
    n = int(n)
    out = np.empty(n, dtype=np.uint32)
    o1 = (ctypes.c_uint32 * 3)()
    o2 = (ctypes.c_uint32 * 3)()
    _lib.check(_lib.lib.prng_kernels_mrg_fill(*st, n, out.ctypes.data if n else None, o1, o2))
    return out, (int(o1[0]), int(o1[1]), int(o1[2])), (int(o2[0]), int(o2[1]), int(o2[2]))


def box_muller(u1, u2):
    """Unit pairs (u1 pre-flipped to (0, 1]) -> standard normal pairs, fp64 (_core.pyx:105)."""
    a = np.ascontiguousarray(u1, dtype=np.float64)
    b = np.ascontiguousarray(u2, dtype=np.float64)
    m = a.shape[0]
    z0 = np.empty(m, dtype=np.float64)
    z1 = np.empty(m, dtype=np.float64)
    if m:
        _lib.check(_lib.lib.prng_kernels_box_muller(a.ctypes.data, b.ctypes.data, m, z0.ctypes.data, z1.ctypes.data))
    return z0, z1
