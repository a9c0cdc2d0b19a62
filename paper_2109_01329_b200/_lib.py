"""ctypes binding of libprng_b200.so (the C ABI in include/prng_b200.h).

There is no fallback: if the shared library is missing or fails to load,
importing this module raises ImportError.  Build it with
``python -c "import __graft_entry__ as g; g.build()"`` or
``make -C paper_2109_01329_b200/csrc``.
"""

from __future__ import annotations

import ctypes
import os
import re
from pathlib import Path

from .errors import Error, InvalidParameter, InvalidRange, UnsupportedEngine

LIB_PATH = Path(os.environ.get("PRNG_B200_LIB", Path(__file__).resolve().parent / "libprng_b200.so"))
HEADER = Path(__file__).resolve().parent.parent / "include" / "prng_b200.h"

PRNG_OK = 0
PRNG_ERR_UNSUPPORTED_ENGINE = -1
PRNG_ERR_INVALID_RANGE = -2
PRNG_ERR_INVALID_PARAMETER = -3
PRNG_ERR_VALUE = -4
PRNG_ERR_CUDA = -5

METHOD_FAST = 0
METHOD_ACCURATE = 1
METHOD_EXACT = 2
METHOD_PRECISE = 3

_u32 = ctypes.c_uint32
_u64 = ctypes.c_uint64
_dbl = ctypes.c_double
_int = ctypes.c_int
_vp = ctypes.c_void_p
_u32p = ctypes.POINTER(ctypes.c_uint32)

_P = [_u32, _u32, _u32p, _u32, _u64]  # k0, k1, ctr[4], lane, n
_M = [_u32p, _u32p, _u64]  # s1[3], s2[3], n

SIGNATURES = {
    "prng_abi_version": ([], _int),
    "prng_last_error": ([], ctypes.c_char_p),
    "prng_philox4x32x10_bits": (_P + [_vp, _vp], _int),
    "prng_philox4x32x10_uniform_f32": (_P + [_dbl, _dbl, _vp, _vp], _int),
    "prng_philox4x32x10_uniform_f64": (_P + [_dbl, _dbl, _vp, _vp], _int),
    "prng_philox4x32x10_gaussian_f32": (_P + [_dbl, _dbl, _int, _vp, _vp], _int),
    "prng_philox4x32x10_gaussian_f64": (_P + [_dbl, _dbl, _vp, _vp], _int),
    "prng_philox4x32x10_gaussian_f64_method": (_P + [_dbl, _dbl, _int, _vp, _vp], _int),
    "prng_philox4x32x10_lognormal_f32": (_P + [_dbl, _dbl, _dbl, _dbl, _int, _vp, _vp], _int),
    "prng_philox4x32x10_lognormal_f64": (_P + [_dbl, _dbl, _dbl, _dbl, _vp, _vp], _int),
    "prng_mrg32k3a_bits": (_M + [_vp, _vp], _int),
    "prng_mrg32k3a_uniform_f32": (_M + [_dbl, _dbl, _vp, _vp], _int),
    "prng_mrg32k3a_uniform_f64": (_M + [_dbl, _dbl, _vp, _vp], _int),
    "prng_mrg32k3a_gaussian_f32": (_M + [_dbl, _dbl, _int, _vp, _vp], _int),
    "prng_mrg32k3a_gaussian_f64": (_M + [_dbl, _dbl, _vp, _vp], _int),
    "prng_mrg32k3a_gaussian_f64_method": (_M + [_dbl, _dbl, _int, _vp, _vp], _int),
    "prng_mrg32k3a_lognormal_f32": (_M + [_dbl, _dbl, _dbl, _dbl, _int, _vp, _vp], _int),
    "prng_mrg32k3a_lognormal_f64": (_M + [_dbl, _dbl, _dbl, _dbl, _vp, _vp], _int),
    "prng_mrg32k3a_skip_ahead": ([_u32p, _u32p, _u64, _u64, _u32p, _u32p], _int),
    "prng_range_transform_f32": ([_vp, _u64, _dbl, _dbl, _vp], _int),
    "prng_range_transform_f64": ([_vp, _u64, _dbl, _dbl, _vp], _int),
    "prng_words_to_unit_f32": ([_vp, _u64, _vp, _vp], _int),
    "prng_words_to_unit_f64": ([_vp, _u64, _vp, _vp], _int),
    "prng_gaussian_from_words_f32": ([_vp, _u64, _dbl, _dbl, _int, _vp, _vp], _int),
    "prng_gaussian_from_words_f64": ([_vp, _u64, _dbl, _dbl, _vp, _vp], _int),
    "prng_gaussian_from_words_f64_method": ([_vp, _u64, _dbl, _dbl, _int, _vp, _vp], _int),
    "prng_exact_tables_prepare": ([], _int),
    "prng_exact_tables_host": ([ctypes.POINTER(ctypes.POINTER(ctypes.c_double))] * 2, _int),
    "prng_exact_tables_bounds": ([ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint64)], _int),
    "prng_philox4x32x10_uniform_f32_segments": ([_u32, _u32, _vp, _u32, _u64, _dbl, _dbl, _vp, _vp], _int),
    "prng_calo_hits": ([_vp, _vp, _u32, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _int),
    "prng_calo_deposit_scratch_bytes": ([_u64, _u32], ctypes.c_size_t),
    "prng_calo_deposit": ([_vp, _vp, _u64, _vp, _u32, _u32, _vp, ctypes.c_size_t, _vp, _vp, _vp, _vp], _int),
    "prng_kernels_philox_fill": ([_u32] * 7 + [_u64, _vp], _int),
    "prng_kernels_mrg_fill": ([_u32] * 6 + [_u64, _vp, _u32p, _u32p], _int),
    "prng_kernels_box_muller": ([_vp, _vp, _u64, _vp, _vp], _int),
    "prng_diag_write_probe": ([_vp, _u64, _vp], _int),
}


def header_symbols(path: Path = HEADER):
    """Function names declared in include/prng_b200.h."""
    text = path.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char \*)\s*(prng_\w+)\s*\(", text, re.M)))


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"libprng_b200.so not found at {LIB_PATH}; build it (make -C paper_2109_01329_b200/csrc). "
            "There is no CPU fallback."
        )
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, (args, res) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()


class CudaError(Error, RuntimeError):
    """CUDA runtime failure inside libprng_b200 (PRNG_ERR_CUDA)."""


_ERRORS = {
    PRNG_ERR_UNSUPPORTED_ENGINE: UnsupportedEngine,
    PRNG_ERR_INVALID_RANGE: InvalidRange,
    PRNG_ERR_INVALID_PARAMETER: InvalidParameter,
    PRNG_ERR_VALUE: ValueError,
    PRNG_ERR_CUDA: CudaError,
}


def check(rc: int) -> None:
    """Raise the reference exception type matching a negative status."""
    if rc == PRNG_OK:
        return
    msg = (lib.prng_last_error() or b"").decode(errors="replace")
    raise _ERRORS.get(rc, Error)(msg or f"libprng_b200 status {rc}")


def u32_array(values):
    arr = (ctypes.c_uint32 * len(values))(*[int(v) & 0xFFFFFFFF for v in values])
    return arr
