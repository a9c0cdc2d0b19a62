# portarng/_kernels/_cuda.py -- CUDA kernel core via libprng_b200.so
# (the ctypes stub of INTEGRATION.md §1, byte for byte; staged into the
# reference copy under baseline/_ref by baseline/stage_ref.sh)
import ctypes, os
import numpy as np

IMPL = "cuda"
_lib = ctypes.CDLL(os.environ.get("PRNG_B200_LIB", "libprng_b200.so"))
_u32, _u64, _vp = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_void_p
_lib.prng_kernels_philox_fill.argtypes = [_u32] * 7 + [_u64, _vp]
_lib.prng_kernels_mrg_fill.argtypes = [_u32] * 6 + [_u64, _vp, ctypes.POINTER(_u32), ctypes.POINTER(_u32)]
_lib.prng_kernels_box_muller.argtypes = [_vp, _vp, _u64, _vp, _vp]
_lib.prng_last_error.restype = ctypes.c_char_p

def _check(rc):
    if rc:
        raise RuntimeError(_lib.prng_last_error().decode())

def philox_fill(k0, k1, b0, b1, b2, b3, offset, n):          # _core.pyx:42
    out = np.empty(n, dtype=np.uint32)
    if n:
        _check(_lib.prng_kernels_philox_fill(k0, k1, b0, b1, b2, b3, offset, n, out.ctypes.data))
    return out

def mrg_fill(s10, s11, s12, s20, s21, s22, n):                # _core.pyx:74
    out = np.empty(n, dtype=np.uint32)
    o1, o2 = (_u32 * 3)(), (_u32 * 3)()
    _check(_lib.prng_kernels_mrg_fill(s10, s11, s12, s20, s21, s22, n, out.ctypes.data if n else None, o1, o2))
    return out, tuple(o1), tuple(o2)

def box_muller(u1, u2):                                        # _core.pyx:105
    a = np.ascontiguousarray(u1, dtype=np.float64)
    b = np.ascontiguousarray(u2, dtype=np.float64)
    z0, z1 = np.empty_like(a), np.empty_like(a)
    if len(a):
        _check(_lib.prng_kernels_box_muller(a.ctypes.data, b.ctypes.data, len(a), z0.ctypes.data, z1.ctypes.data))
    return z0, z1
