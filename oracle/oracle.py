"""CPU oracle for the RNG hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker.
The product package (paper_2109_01329_b200) never imports it; its CUDA path
fails loudly when the extension is missing.

Two independent CPU routes live here:

* ``liboracle.so`` (oracle.c): a plain-C restatement of the reference kernel
  core, used for everything (parity checks, the "port" CPU baseline).
* ``oracle/_ref/_core*.so``: the reference's own Cython core compiled from
  /root/reference by build_ref.sh, used to pin the restatement and as the
  "reference" CPU baseline when present.

Stream semantics (positions, pairing, precision) follow the reference:
engine.py:125-146 (word positions), distributions.py:78-153 (unit map,
affine, Box-Muller), rngburn.py:62-91 (chunked kernels).  The post-processing
on top of the raw words is written with numpy exactly as the reference
writes it, so numpy's own rounding rules (NEP-50 weak scalars) apply.
"""

from __future__ import annotations

import ctypes
import importlib.util
import os
import subprocess
import sys
from pathlib import Path
from typing import Optional, Tuple

import numpy as np

HERE = Path(__file__).resolve().parent
MASK32 = 0xFFFFFFFF
MASK64 = (1 << 64) - 1
MRG_M1 = 4294967087
MRG_M2 = 4294944443
UNIT_SCALE = 2.0 ** -24

_u32p = ctypes.POINTER(ctypes.c_uint32)
_f32p = ctypes.POINTER(ctypes.c_float)
_f64p = ctypes.POINTER(ctypes.c_double)
_lib = None


def build() -> Path:
    """Compile liboracle.so with oracle/Makefile (gcc)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return HERE / "liboracle.so"


def lib():
    global _lib
    if _lib is None:
        path = HERE / "liboracle.so"
        if not path.exists():
            build()
        L = ctypes.CDLL(str(path))
        L.oracle_philox_block.argtypes = [ctypes.c_uint32, ctypes.c_uint32, _u32p, _u32p]
        L.oracle_philox_fill.argtypes = [ctypes.c_uint32, ctypes.c_uint32, _u32p, ctypes.c_uint32,
                                         ctypes.c_uint64, _u32p]
        L.oracle_mrg_fill.argtypes = [_u32p, _u32p, ctypes.c_uint64, _u32p]
        L.oracle_mrg_skip.argtypes = [_u32p, _u32p, ctypes.c_uint64, ctypes.c_uint64]
        L.oracle_box_muller.argtypes = [_f64p, _f64p, ctypes.c_uint64, _f64p, _f64p]
        L.oracle_gaussian_f64.argtypes = [_u32p, ctypes.c_uint64, ctypes.c_double, ctypes.c_double, _f64p]
        L.oracle_gaussian_f32.argtypes = [_u32p, ctypes.c_uint64, ctypes.c_double, ctypes.c_double, _f32p]
        L.oracle_lognormal_f64.argtypes = [_u32p, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, _f64p]
        L.oracle_lognormal_f32.argtypes = [_u32p, ctypes.c_uint64, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, _f32p]
        L.oracle_range_f32.argtypes = [_f32p, ctypes.c_uint64, ctypes.c_double, ctypes.c_double]
        L.oracle_range_f64.argtypes = [_f64p, ctypes.c_uint64, ctypes.c_double, ctypes.c_double]
        for name in ("oracle_philox_block", "oracle_philox_fill", "oracle_mrg_fill", "oracle_mrg_skip",
                     "oracle_box_muller", "oracle_gaussian_f64", "oracle_gaussian_f32",
                     "oracle_lognormal_f64", "oracle_lognormal_f32", "oracle_range_f32", "oracle_range_f64"):
            getattr(L, name).restype = None
        _lib = L
    return _lib


def _p(arr, typ):
    return arr.ctypes.data_as(typ)


def ref_core():
    """The reference's compiled Cython core (oracle/_ref), or None if not built."""
    d = HERE / "_ref"
    if not d.is_dir():
        return None
    for f in sorted(d.iterdir()):
        if f.name.startswith("_core") and f.suffix == ".so":
            spec = importlib.util.spec_from_file_location("_core", f)
            mod = importlib.util.module_from_spec(spec)
            try:
                spec.loader.exec_module(mod)
            except ImportError:
                return None
            return mod
    return None


# ---------------------------------------------------------------- engines


def philox_block(key: Tuple[int, int], ctr: Tuple[int, int, int, int]) -> Tuple[int, ...]:
    """engine.py:86-103."""
    c = np.array(ctr, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox_block(key[0] & MASK32, key[1] & MASK32, _p(c, _u32p), _p(out, _u32p))
    return tuple(int(x) for x in out)


def philox_fill(k0, k1, b0, b1, b2, b3, offset, n) -> np.ndarray:
    """Same signature and result as the reference kernel `philox_fill` (_core.pyx:42)."""
    out = np.empty(n, dtype=np.uint32)
    blk = np.array([b0, b1, b2, b3], dtype=np.uint32)
    if n:
        lib().oracle_philox_fill(k0, k1, _p(blk, _u32p), offset, n, _p(out, _u32p))
    return out


def philox_words(key: Tuple[int, int], position: int, n: int) -> np.ndarray:
    """n stream words starting at absolute word `position` (engine.py:212-226)."""
    block, lane = divmod(position % (1 << 130), 4)
    block %= 1 << 128
    b = [(block >> (32 * i)) & MASK32 for i in range(4)]
    return philox_fill(key[0], key[1], *b, lane, n)


def mrg_fill(s10, s11, s12, s20, s21, s22, n):
    """Same signature and result as the reference kernel `mrg_fill` (_core.pyx:74)."""
    s1 = np.array([s10, s11, s12], dtype=np.uint32)
    s2 = np.array([s20, s21, s22], dtype=np.uint32)
    out = np.empty(n, dtype=np.uint32)
    lib().oracle_mrg_fill(_p(s1, _u32p), _p(s2, _u32p), n, _p(out, _u32p))
    return out, tuple(int(x) for x in s1), tuple(int(x) for x in s2)


def mrg_skip(s1, s2, k: int):
    """State after k sequential steps (extension a19; A^k s mod m)."""
    a = np.array(s1, dtype=np.uint32)
    b = np.array(s2, dtype=np.uint32)
    lib().oracle_mrg_skip(_p(a, _u32p), _p(b, _u32p), k & MASK64, (k >> 64) & MASK64)
    return tuple(int(x) for x in a), tuple(int(x) for x in b)


def box_muller(u1: np.ndarray, u2: np.ndarray):
    """_core.pyx:105-122 (libm, fp64)."""
    a = np.ascontiguousarray(u1, dtype=np.float64)
    b = np.ascontiguousarray(u2, dtype=np.float64)
    z0 = np.empty_like(a)
    z1 = np.empty_like(a)
    if len(a):
        lib().oracle_box_muller(_p(a, _f64p), _p(b, _f64p), len(a), _p(z0, _f64p), _p(z1, _f64p))
    return z0, z1


def seed_philox(seed: int) -> Tuple[int, int]:
    """engine.py:114-116: key = (seed lo32, seed hi32)."""
    seed &= MASK64
    return (seed & MASK32, seed >> 32)


def seed_mrg(seed: int):
    """engine.py:117-121: v = seed mod m2 (0 -> 12345)."""
    v = (seed & MASK64) % MRG_M2
    if v == 0:
        v = 12345
    return (v, v, v), (v, v, v)


# ------------------------------------------------------------ distributions


def words_to_unit(words: np.ndarray, precision: str = "fp32") -> np.ndarray:
    """distributions.py:83-87."""
    dtype = np.float32 if precision == "fp32" else np.float64
    return (words >> np.uint32(8)).astype(dtype) * dtype(UNIT_SCALE)


def range_transform(values: np.ndarray, lo: float, hi: float) -> np.ndarray:
    """distributions.py:98-104 (numpy NEP-50 weak-scalar rounding, in place)."""
    values *= hi - lo
    values += lo
    return values


def gaussian_from_words(words: np.ndarray, mean: float, stddev: float, n: int, precision: str = "fp32"):
    """distributions.py:116-131 with box_muller from libm (as the reference core)."""
    u1 = (words[0::2] >> np.uint32(8)).astype(np.float64) * UNIT_SCALE
    u2 = (words[1::2] >> np.uint32(8)).astype(np.float64) * UNIT_SCALE
    z0, z1 = box_muller(1.0 - u1, u2)
    z = np.empty(2 * len(u1), dtype=np.float64)
    z[0::2] = z0
    z[1::2] = z1
    z *= stddev
    z += mean
    return z[:n].astype(np.float32 if precision == "fp32" else np.float64)


def lognormal_from_words(words: np.ndarray, m: float, s: float, n: int, precision: str = "fp32",
                         displ: float = 0.0, scale: float = 1.0):
    """Lognormal extension (a18): exp of the fp64 gaussian, then scale/displ, then cast."""
    out = np.empty(n, dtype=np.float64)
    w = np.ascontiguousarray(words, dtype=np.uint32)
    if n:
        lib().oracle_lognormal_f64(_p(w, _u32p), n, m, s, displ, scale, _p(out, _f64p))
    return out.astype(np.float32 if precision == "fp32" else np.float64)


# ------------------------------------------------ whole-request generators


def stream_words(engine: str, state, n: int) -> np.ndarray:
    """n words from an engine state given as ('philox', key, position) or ('mrg', s1, s2)."""
    if engine == "philox":
        key, pos = state
        return philox_words(key, pos, n)
    s1, s2 = state
    return mrg_fill(*s1, *s2, n)[0]


def generate(engine: str, state, dist: str, n: int, precision: str = "fp32", a: float = 0.0,
             b: float = 1.0, displ: float = 0.0, scale: float = 1.0) -> np.ndarray:
    """Reference result of one fused request.

    dist: 'bits' (uint32 words), 'uniform' on [a, b) (fill_uniform_unit +
    range_transform), 'gaussian' (mean a, stddev b; fill_gaussian),
    'lognormal' (m a, s b; extension).
    """
    if dist == "bits":
        return stream_words(engine, state, n)
    if dist == "uniform":
        v = words_to_unit(stream_words(engine, state, n), precision)
        return range_transform(v, a, b)
    nwords = 2 * ((n + 1) // 2)
    words = stream_words(engine, state, nwords)
    if dist == "gaussian":
        if n == 0:
            return np.empty(0, dtype=np.float32 if precision == "fp32" else np.float64)
        return gaussian_from_words(words, a, b, n, precision)
    if dist == "lognormal":
        return lognormal_from_words(words, a, b, n, precision, displ, scale)
    raise ValueError(dist)


def sha16(arr: np.ndarray) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()[:16]
