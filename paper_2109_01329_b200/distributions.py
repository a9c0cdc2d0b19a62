"""Distribution requests and the fused device generators.

Mirrors pkg/src/portarng/distributions.py (names, validation, word
accounting, precision rules) and adds the oneMKL-style entry point
``generate(distribution, engine_state, n, out)`` the north star names, plus
``UniformBits`` and ``Lognormal``.

Every generator is ONE kernel launch (libprng_b200.so) that draws the words,
applies the distribution transform and writes each sample to HBM once; the
reference's separate generate -> words_to_unit -> range_transform passes
(rngburn.py:142-147) are fused.  Outputs live on the GPU as torch tensors.

Results vs the reference:
  * uniform_bits, uniform fp32/fp64 on [a, b): bit-exact;
  * gaussian/lognormal fp64, and fp32 with method="accurate": fp64 math on
    the device (CUDA libdevice log/sincos/exp vs glibc), a few fp64 ulps;
  * gaussian/lognormal fp32 with method="fast" (default): fp32 SFU lg2 /
    sqrt (series near u1 = 0), sin/cos from the nearest point of a table,
    ex2: |err| <= 2^-20 * stddev * max(1, |z|), <= 8 ulp for |z| >= 1;
  * method="precise" (fp32): table log + centred sin/cos with the x^2 term,
    within 5 ulp of the reference for every input (lognormal: 5 ulp *
    max(1, |ln x|)), ~85% of "fast"'s throughput;
  * gaussian fp32/fp64 with method="exact": bit-identical to the reference
    (device log / sin / cos corrected to the host libm by per-input ulp
    deltas over their whole 2^24-point input domains, csrc/common.cuh
    box_muller_exact).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Tuple, Union

from . import _lib
from .engine import (
    EngineKind,
    EngineState,
    Mrg32k3a,
    Mrg32k3aState,
    Philox4x32x10,
    PhiloxState,
    _out_tensor,
    _stream_handle,
    _torch,
    advance,
    generate_words,
    mrg_args,
    philox_args,
)
from .errors import InvalidParameter, InvalidRange, UnsupportedEngine

_UNIT_SCALE = 2.0 ** -24
_PRECISIONS = ("fp32", "fp64")
_METHODS = {"fast": _lib.METHOD_FAST, "accurate": _lib.METHOD_ACCURATE, "exact": _lib.METHOD_EXACT,
            "precise": _lib.METHOD_PRECISE}


def _check_precision(precision: str) -> None:
    if precision not in _PRECISIONS:
        raise InvalidParameter(f"precision must be fp32 or fp64, got {precision!r}")


def _check_method(method: str, exact_ok: bool = True) -> None:
    if method not in _METHODS or (method == "exact" and not exact_ok):
        allowed = "'fast', 'precise', 'accurate' or 'exact'" if exact_ok else "'fast', 'precise' or 'accurate'"
        raise InvalidParameter(f"method must be {allowed}, got {method!r}")


def _dtype(precision: str):
    torch = _torch()
    return torch.float32 if precision == "fp32" else torch.float64


@dataclass(frozen=True)
class Uniform:
    """Uniform draw request over [lo, hi) (distributions.py:38-49)."""

    lo: float
    hi: float
    precision: str = "fp32"

    def __post_init__(self):
        if not (math.isfinite(self.lo) and math.isfinite(self.hi)) or self.lo >= self.hi:
            raise InvalidRange(f"uniform range requires finite lo < hi, got [{self.lo}, {self.hi})")
        _check_precision(self.precision)


@dataclass(frozen=True)
class Gaussian:
    """Normal draw request (distributions.py:52-63); Box-Muller pairs."""

    mean: float
    stddev: float
    precision: str = "fp32"
    method: str = "fast"

    def __post_init__(self):
        if not math.isfinite(self.mean) or not math.isfinite(self.stddev) or self.stddev <= 0:
            raise InvalidParameter(f"gaussian requires finite mean and stddev > 0, got ({self.mean}, {self.stddev})")
        _check_precision(self.precision)
        _check_method(self.method)


@dataclass(frozen=True)
class Lognormal:
    """Lognormal request x = displ + scale * exp(m + s z) (oneMKL lognormal;
    absent from the reference)."""

    m: float = 0.0
    s: float = 1.0
    displ: float = 0.0
    scale: float = 1.0
    precision: str = "fp32"
    method: str = "fast"

    def __post_init__(self):
        vals = (self.m, self.s, self.displ, self.scale)
        if not all(math.isfinite(v) for v in vals) or self.s <= 0 or self.scale <= 0:
            raise InvalidParameter(f"lognormal requires finite m, s > 0, finite displ, scale > 0, got {vals}")
        _check_precision(self.precision)
        _check_method(self.method, exact_ok=False)


@dataclass(frozen=True)
class UniformBits:
    """Raw engine words: oneMKL uniform_bits<uint32> (bits=32, one word per
    sample) or uniform_bits<uint64> (bits=64: sample i = word 2i | word
    (2i+1) << 32, i.e. the 32-bit stream read as little-endian 64-bit
    values; two words per sample)."""

    bits: int = 32

    def __post_init__(self):
        if self.bits not in (32, 64):
            raise InvalidParameter(f"uniform_bits width must be 32 or 64, got {self.bits!r}")


DistributionSpec = Union[Uniform, Gaussian, Lognormal, UniformBits]


@dataclass
class RandomBlock:
    """A generated batch (distributions.py:69-75); `values` is a CUDA tensor."""

    values: object
    count: int
    precision: str = "fp32"


def words_consumed(spec: DistributionSpec, n: int) -> int:
    """Stream words a request of n samples consumes (distributions.py:146-149)."""
    if isinstance(spec, (Gaussian, Lognormal)):
        return 2 * ((n + 1) // 2)
    if isinstance(spec, UniformBits) and spec.bits == 64:
        return 2 * n
    return n


def word_to_unit(w: int) -> float:
    """distributions.py:78-80 (scalar helper; exact arithmetic)."""
    return (w >> 8) * _UNIT_SCALE


def words_to_unit(words, precision: str = "fp32", out=None, stream=None):
    """Device words -> unit values, (w >> 8) * 2**-24 (distributions.py:83-87)."""
    _check_precision(precision)
    n = words.numel()
    out = _out_tensor(out, n, _dtype(precision), words.device)
    fn = _lib.lib.prng_words_to_unit_f32 if precision == "fp32" else _lib.lib.prng_words_to_unit_f64
    _lib.check(fn(words.data_ptr(), n, out.data_ptr(), _stream_handle(stream, out.device)))
    return out[:n]


def gaussian_from_words(words, mean: float, stddev: float, n: int, precision: str = "fp32",
                        method: str = "fast", out=None, stream=None):
    """distributions.py:116-131 on device words (2*ceil(n/2) of them)."""
    _check_precision(precision)
    _check_method(method)
    if words.numel() < 2 * ((n + 1) // 2):
        raise InvalidParameter("need 2*ceil(n/2) words")
    out = _out_tensor(out, n, _dtype(precision), words.device)
    s = _stream_handle(stream, out.device)
    if precision == "fp32":
        rc = _lib.lib.prng_gaussian_from_words_f32(words.data_ptr(), n, mean, stddev, _METHODS[method],
                                                   out.data_ptr(), s)
    else:
        rc = _lib.lib.prng_gaussian_from_words_f64_method(words.data_ptr(), n, mean, stddev, _METHODS[method],
                                                          out.data_ptr(), s)
    _lib.check(rc)
    return out[:n]


_PREFIX = {EngineKind.PHILOX4X32X10: "prng_philox4x32x10_", EngineKind.MRG32K3A: "prng_mrg32k3a_"}
_FN_CACHE = {}


def _entry(kind: EngineKind, spec: DistributionSpec):
    """The C-ABI function and the distribution arguments for one request shape."""
    if isinstance(spec, UniformBits):
        name, tail = "bits", ()
    elif isinstance(spec, Uniform):
        name, tail = "uniform_" + ("f32" if spec.precision == "fp32" else "f64"), (spec.lo, spec.hi)
    elif isinstance(spec, Gaussian):
        if spec.precision == "fp32":
            name, tail = "gaussian_f32", (spec.mean, spec.stddev, _METHODS[spec.method])
        else:
            name, tail = "gaussian_f64_method", (spec.mean, spec.stddev, _METHODS[spec.method])
    elif isinstance(spec, Lognormal):
        if spec.precision == "fp32":
            name, tail = "lognormal_f32", (spec.m, spec.s, spec.displ, spec.scale, _METHODS[spec.method])
        else:
            name, tail = "lognormal_f64", (spec.m, spec.s, spec.displ, spec.scale)
    else:
        raise InvalidParameter(f"unknown distribution {spec!r}")
    key = (kind, name)
    fn = _FN_CACHE.get(key)
    if fn is None:
        fn = _FN_CACHE[key] = getattr(_lib.lib, _PREFIX[kind] + name)
    return fn, tail


def _launch(spec: DistributionSpec, state, n: int, ptr: int, s) -> None:
    if isinstance(state, (Philox4x32x10, Mrg32k3a)):
        kind, head = state.kind, state.launch_args()
    elif isinstance(state, PhiloxState):
        kind, head = EngineKind.PHILOX4X32X10, philox_args(state)
    elif isinstance(state, Mrg32k3aState):
        kind, head = EngineKind.MRG32K3A, mrg_args(state)
    else:
        raise UnsupportedEngine(f"unknown engine state: {type(state).__name__}")
    fn, tail = _entry(kind, spec)
    # uniform_bits<uint64>: the 2n-word stream written as little-endian pairs
    _lib.check(fn(*head, words_consumed(spec, n) if isinstance(spec, UniformBits) else n, *tail, ptr, s))


def out_dtype(spec: DistributionSpec):
    torch = _torch()
    if isinstance(spec, UniformBits):
        return torch.uint64 if spec.bits == 64 else torch.uint32
    return _dtype(spec.precision)


def generate(distribution: DistributionSpec, engine: EngineState, n: int, out=None, stream=None):
    """oneMKL-style generate(distr, engine, n, r): n samples into `out`
    (a CUDA tensor; allocated if None) on `stream`.  Returns
    (advanced_engine_state, out[:n]).  One fused kernel launch."""
    if n < 0:
        raise InvalidParameter("count must be non-negative")
    out = _out_tensor(out, n, out_dtype(distribution))
    if n:
        _launch(distribution, engine, n, out.data_ptr(), _stream_handle(stream, out.device))
    if isinstance(engine, (Philox4x32x10, Mrg32k3a)):
        new_state = engine.skip_ahead(words_consumed(distribution, n))  # oneMKL engines advance in place
    else:
        new_state = advance(engine, words_consumed(distribution, n))
    return new_state, (out if out.numel() == n else out[:n])


def fill_uniform_unit(state: EngineState, n: int, precision: str = "fp32", out=None, stream=None):
    """distributions.py:90-95: n unit uniforms; state advances n words."""
    if n < 0:
        raise InvalidParameter("count must be non-negative")
    _check_precision(precision)
    state, values = generate(Uniform(0.0, 1.0, precision), state, n, out, stream)
    return state, RandomBlock(values=values, count=n, precision=precision)


def fill_uniform(state: EngineState, n: int, lo: float, hi: float, precision: str = "fp32", out=None,
                 stream=None):
    """Fused fill_uniform_unit + range_transform (one pass, bit-identical)."""
    state, values = generate(Uniform(lo, hi, precision), state, n, out, stream)
    return state, RandomBlock(values=values, count=n, precision=precision)


def range_transform(block: RandomBlock, lo: float, hi: float, stream=None) -> RandomBlock:
    """distributions.py:98-104: in-place affine map of unit values onto [lo, hi)."""
    if not (math.isfinite(lo) and math.isfinite(hi)) or lo >= hi:
        raise InvalidRange(f"range transform requires finite lo < hi, got [{lo}, {hi})")
    v = block.values
    fn = _lib.lib.prng_range_transform_f32 if block.precision == "fp32" else _lib.lib.prng_range_transform_f64
    _lib.check(fn(v.data_ptr(), v.numel(), lo, hi, _stream_handle(stream, v.device)))
    return block


def fill_gaussian(state: EngineState, n: int, mean: float, stddev: float, precision: str = "fp32",
                  out=None, stream=None, method: str = "fast"):
    """distributions.py:134-153: n normals, state advances 2*ceil(n/2) words."""
    if n < 0:
        raise InvalidParameter("count must be non-negative")
    state, values = generate(Gaussian(mean, stddev, precision, method), state, n, out, stream)
    return state, RandomBlock(values=values, count=n, precision=precision)


def fill_lognormal(state: EngineState, n: int, m: float = 0.0, s: float = 1.0, displ: float = 0.0,
                   scale: float = 1.0, precision: str = "fp32", out=None, stream=None, method: str = "fast"):
    """Lognormal extension; state advances 2*ceil(n/2) words."""
    if n < 0:
        raise InvalidParameter("count must be non-negative")
    state, values = generate(Lognormal(m, s, displ, scale, precision, method), state, n, out, stream)
    return state, RandomBlock(values=values, count=n, precision=precision)


def exact_tables_host():
    """The exact method's host tables as numpy views (no copy): log(m 2^-24)
    for m = 1..2^24, and (sin t, cos t) for t = fl(TWO_PI k 2^-24), k < 2^24."""
    import numpy as np

    lp = ctypes.POINTER(ctypes.c_double)()
    sp = ctypes.POINTER(ctypes.c_double)()
    _lib.check(_lib.lib.prng_exact_tables_host(ctypes.byref(lp), ctypes.byref(sp)))
    n = 1 << 24
    log_tab = np.ctypeslib.as_array(lp, shape=(n,))
    sc_tab = np.ctypeslib.as_array(sp, shape=(n, 2))
    return log_tab, sc_tab
