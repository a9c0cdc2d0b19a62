"""Engine states and stream-position bookkeeping (host side of the hot path).

Mirrors pkg/src/portarng/engine.py: same names, state types, seed mapping
and error behaviour.  What changes:

* every word is produced on the GPU (libprng_b200.so) -- `generate_words`
  returns a device tensor, and even the scalar `philox_block` / `next_word`
  helpers run on the device: there is no CPU compute path;
* `skip_ahead` also works for MRG32k3a (matrix-power jump-ahead, computed
  by the C library's host code; the reference raises UnsupportedEngine,
  engine.py:201-202).

The state bookkeeping itself (128-bit positions, lanes, windows) is plain
integer arithmetic on the host, exactly as in the reference
(engine.py:125-146, 194-209).
"""

from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass
from typing import Optional, Tuple, Union

from . import _lib
from .errors import InvalidParameter, UnsupportedEngine

MASK32 = 0xFFFFFFFF
MASK64 = 0xFFFFFFFFFFFFFFFF
MASK128 = (1 << 128) - 1

PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85
PHILOX_ROUNDS = 10

MRG_M1 = 4294967087
MRG_M2 = 4294944443
MRG_A12 = 1403580
MRG_A13N = 810728
MRG_A21 = 527612
MRG_A23N = 1370589
MRG_DEFAULT_SEED = 12345


class EngineKind(enum.Enum):
    PHILOX4X32X10 = "philox"
    MRG32K3A = "mrg32k3a"


@dataclass(frozen=True)
class PhiloxState:
    """Philox stream position (engine.py:57-72): key pair, 128-bit counter of
    the next block, lane_index in 0..4 (4 = no block buffered)."""

    key: Tuple[int, int]
    counter: Tuple[int, int, int, int]
    lane_index: int
    cached_block: Optional[Tuple[int, int, int, int]] = None


@dataclass(frozen=True)
class Mrg32k3aState:
    """MRG32k3a recurrence windows (engine.py:75-80)."""

    s1: Tuple[int, int, int]
    s2: Tuple[int, int, int]


EngineState = Union[PhiloxState, Mrg32k3aState]


def seed_engine(kind: EngineKind, seed: int) -> EngineState:
    """engine.py:106-122: Philox key = (seed lo32, hi32), counter 0, lane 4;
    MRG32k3a all six components = seed mod m2 (0 -> 12345)."""
    seed &= MASK64
    if kind is EngineKind.PHILOX4X32X10:
        return PhiloxState(key=(seed & MASK32, seed >> 32), counter=(0, 0, 0, 0), lane_index=4)
    if kind is EngineKind.MRG32K3A:
        v = seed % MRG_M2
        if v == 0:
            v = MRG_DEFAULT_SEED
        return Mrg32k3aState(s1=(v, v, v), s2=(v, v, v))
    raise UnsupportedEngine(f"unknown engine kind: {kind!r}")


def _ctr_to_int(counter) -> int:
    return counter[0] | counter[1] << 32 | counter[2] << 64 | counter[3] << 96


def _int_to_ctr(value: int) -> Tuple[int, int, int, int]:
    value &= MASK128
    return (value & MASK32, (value >> 32) & MASK32, (value >> 64) & MASK32, (value >> 96) & MASK32)


def _position(state: PhiloxState) -> int:
    c = _ctr_to_int(state.counter)
    if state.lane_index == 4:
        return 4 * c
    return 4 * ((c - 1) % (1 << 128)) + state.lane_index


def _state_at(key, position: int) -> PhiloxState:
    block, lane = divmod(position, 4)
    if lane == 0:
        return PhiloxState(key=key, counter=_int_to_ctr(block), lane_index=4)
    return PhiloxState(key=key, counter=_int_to_ctr(block + 1), lane_index=lane)


def stream_position(state: PhiloxState) -> int:
    """engine.py:183-191 (Philox only)."""
    if not isinstance(state, PhiloxState):
        raise UnsupportedEngine("stream positions are defined for Philox states")
    return _position(state)


def philox_args(state: PhiloxState):
    """(k0, k1, ctr[4], lane) of the next word -- the C-ABI Philox state
    arguments (philox_fill's (k0, k1, b0..b3, offset), engine.py:221-225)."""
    block, lane = divmod(_position(state), 4)
    return state.key[0] & MASK32, state.key[1] & MASK32, _lib.u32_array(_int_to_ctr(block)), lane


def mrg_args(state: Mrg32k3aState):
    return _lib.u32_array(state.s1), _lib.u32_array(state.s2)


def _mrg_skip(state: Mrg32k3aState, n: int) -> Mrg32k3aState:
    s1, s2 = mrg_args(state)
    o1 = (ctypes.c_uint32 * 3)()
    o2 = (ctypes.c_uint32 * 3)()
    _lib.check(_lib.lib.prng_mrg32k3a_skip_ahead(s1, s2, n & MASK64, (n >> 64) & MASK64, o1, o2))
    return Mrg32k3aState(tuple(o1), tuple(o2))


def skip_ahead(state: EngineState, n: int) -> EngineState:
    """Advance by n words as if drawn and discarded (engine.py:194-209).

    Philox: O(1) counter arithmetic.  MRG32k3a: A^n s mod m (extension; the
    reference raises UnsupportedEngine here).  n < 0 raises ValueError; n == 0
    returns the same object.
    """
    if not isinstance(state, (PhiloxState, Mrg32k3aState)):
        raise UnsupportedEngine(f"unknown engine state: {type(state).__name__}")
    if n < 0:
        raise ValueError("skip count must be non-negative")
    if n == 0:
        return state
    if isinstance(state, Mrg32k3aState):
        return _mrg_skip(state, n)
    return _state_at(state.key, _position(state) + n)


def advance(state: EngineState, nwords: int) -> EngineState:
    """State after a request that consumed `nwords` words (no identity shortcut)."""
    return skip_ahead(state, nwords) if nwords else state


def _torch():
    import torch

    return torch


_RAW_STREAM = None


def _stream_handle(stream, device=None):
    """cudaStream_t for a launch: `stream` (torch Stream or raw handle), else
    the current torch stream of `device` (of the current device if None)."""
    global _RAW_STREAM
    if stream is None:
        torch = _torch()
        if _RAW_STREAM is None:
            # torch's own raw-handle query: no Stream object per launch (~2 us saved)
            _RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", False)
        idx = None
        if device is not None:
            dev = device if isinstance(device, torch.device) else torch.device(device)
            if dev.type == "cuda":
                idx = dev.index
        if _RAW_STREAM:
            return _RAW_STREAM(torch.cuda.current_device() if idx is None else idx)
        return torch.cuda.current_stream(idx).cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _out_tensor(out, n, dtype, device=None):
    torch = _torch()
    if out is None:
        return torch.empty(n, dtype=dtype, device=device if device is not None else "cuda")
    if out.dtype != dtype:
        raise InvalidParameter(f"out has dtype {out.dtype}, expected {dtype}")
    if not out.is_cuda and not out.is_pinned():
        raise InvalidParameter("out must be a CUDA tensor or pinned host memory")
    if not out.is_contiguous() or out.numel() < n:
        raise InvalidParameter(f"out must be contiguous with at least {n} elements")
    return out


def generate_words(state: EngineState, n: int, out=None, stream=None):
    """n raw 32-bit words on the device; equivalent to n `next_word` calls
    (engine.py:212-232).  Returns (new_state, uint32 CUDA tensor)."""
    if n < 0:
        raise ValueError("word count must be non-negative")
    if not isinstance(state, (PhiloxState, Mrg32k3aState)):
        raise UnsupportedEngine(f"unknown engine state: {type(state).__name__}")
    torch = _torch()
    out = _out_tensor(out, n, torch.uint32)
    if n:
        s = _stream_handle(stream, out.device)
        if isinstance(state, PhiloxState):
            k0, k1, ctr, lane = philox_args(state)
            _lib.check(_lib.lib.prng_philox4x32x10_bits(k0, k1, ctr, lane, n, out.data_ptr(), s))
        else:
            s1, s2 = mrg_args(state)
            _lib.check(_lib.lib.prng_mrg32k3a_bits(s1, s2, n, out.data_ptr(), s))
    if n == 0:
        return state, out[:0]
    return advance(state, n), out[:n] if out.numel() != n else out


def philox_block(key: Tuple[int, int], counter: Tuple[int, int, int, int]) -> Tuple[int, int, int, int]:
    """One Philox4x32-10 block (engine.py:86-103), computed on the device."""
    state = PhiloxState(key=(key[0] & MASK32, key[1] & MASK32), counter=tuple(counter), lane_index=4)
    _, words = generate_words(state, 4)
    return tuple(int(x) for x in words.cpu().tolist())


def next_word(state: EngineState):
    """Draw one word (engine.py:149-175); behavioural helper, device-computed."""
    if isinstance(state, PhiloxState):
        if state.lane_index == 4:
            block = philox_block(state.key, state.counter)
            ctr = _int_to_ctr(_ctr_to_int(state.counter) + 1)
            return PhiloxState(state.key, ctr, 1, block), block[0]
        block = state.cached_block
        if block is None:
            block = philox_block(state.key, _int_to_ctr(_ctr_to_int(state.counter) - 1))
        word = block[state.lane_index]
        return PhiloxState(state.key, state.counter, state.lane_index + 1, block), word
    if isinstance(state, Mrg32k3aState):
        new, words = generate_words(state, 1)
        return new, int(words.cpu()[0])
    raise UnsupportedEngine(f"unknown engine state: {type(state).__name__}")


def mrg_unit(z: int) -> float:
    """engine.py:178-180."""
    return z / (MRG_M1 + 1)


class Philox4x32x10:
    """oneMKL-style stateful engine (`oneapi::mkl::rng::philox4x32x10(queue,
    seed)`, the interface the paper extends).

    Holds the key and the absolute word position; `generate(distr, engine,
    n, out)` advances it in place.  `state` / `from_state` convert to and
    from the reference's immutable PhiloxState (engine.py:57-72).
    """

    kind = EngineKind.PHILOX4X32X10

    def __init__(self, seed: int = 0, offset: int = 0):
        st = seed_engine(EngineKind.PHILOX4X32X10, seed)
        self.key = st.key
        self.position = 0
        self._ctr = (ctypes.c_uint32 * 4)()
        if offset:
            self.skip_ahead(offset)

    @classmethod
    def from_state(cls, state: PhiloxState) -> "Philox4x32x10":
        eng = cls.__new__(cls)
        eng.key = state.key
        eng.position = _position(state)
        eng._ctr = (ctypes.c_uint32 * 4)()
        return eng

    @property
    def state(self) -> PhiloxState:
        return _state_at(self.key, self.position)

    def skip_ahead(self, n: int) -> "Philox4x32x10":
        if n < 0:
            raise ValueError("skip count must be non-negative")
        self.position = (self.position + n) % (1 << 130)
        return self

    def launch_args(self):
        blk = self.position >> 2
        c = self._ctr
        c[0] = blk & MASK32
        c[1] = (blk >> 32) & MASK32
        c[2] = (blk >> 64) & MASK32
        c[3] = (blk >> 96) & MASK32
        return (self.key[0] & MASK32, self.key[1] & MASK32, c, self.position & 3)


class Mrg32k3a:
    """oneMKL-style stateful MRG32k3a engine (`oneapi::mkl::rng::mrg32k3a`)."""

    kind = EngineKind.MRG32K3A

    def __init__(self, seed: int = 0, offset: int = 0):
        st = seed_engine(EngineKind.MRG32K3A, seed)
        self._set(st.s1, st.s2)
        if offset:
            self.skip_ahead(offset)

    def _set(self, s1, s2):
        self._s1 = _lib.u32_array(s1)
        self._s2 = _lib.u32_array(s2)

    @classmethod
    def from_state(cls, state: Mrg32k3aState) -> "Mrg32k3a":
        eng = cls.__new__(cls)
        eng._set(state.s1, state.s2)
        return eng

    @property
    def state(self) -> Mrg32k3aState:
        return Mrg32k3aState(tuple(self._s1), tuple(self._s2))

    def skip_ahead(self, n: int) -> "Mrg32k3a":
        if n < 0:
            raise ValueError("skip count must be non-negative")
        if n:
            _lib.check(_lib.lib.prng_mrg32k3a_skip_ahead(self._s1, self._s2, n & MASK64, (n >> 64) & MASK64,
                                                         self._s1, self._s2))
        return self

    def launch_args(self):
        return (self._s1, self._s2)


Engine = Union[Philox4x32x10, Mrg32k3a]
