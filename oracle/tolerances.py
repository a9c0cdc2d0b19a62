"""Stated tolerances for the floating-point distributions.

Integer words and uniform fp32/fp64 are compared bit-exactly elsewhere; the
functions here return the per-element allowed |gpu - ref| for gaussian and
lognormal outputs, given the reference (oracle) values.
"""

import numpy as np

# fp32 fast path (logf / sqrtf / sincospif / fmaf): absolute error on the
# standard-normal scale of 2^-19 * max(1, |z|), plus 2 ulp of the output.
GAUSS_F32_FAST_REL = 2.0 ** -19
# fp64 path (CUDA log / sincos / exp vs glibc): 2^-45 on the standard-normal
# scale (a few ulp of |z| <= 5.8), plus 2 ulp of the output.
GAUSS_F64_REL = 2.0 ** -45


def ulp(x, dtype):
    x = np.abs(np.asarray(x, dtype=dtype))
    return np.spacing(x).astype(np.float64)


def gaussian_allowed(ref, mean, stddev, dtype, fast):
    ref64 = np.asarray(ref, dtype=np.float64)
    z = np.abs((ref64 - mean) / stddev)
    rel = GAUSS_F32_FAST_REL if (fast and dtype == np.float32) else GAUSS_F64_REL
    if dtype == np.float32 and not fast:
        # accurate fp32 = fp64 math then one cast: at most 1 ulp from the cast
        return ulp(ref, np.float32)
    return stddev * rel * np.maximum(1.0, z) + 2 * ulp(ref, dtype) + 2 * ulp(mean, dtype)


def lognormal_allowed(ref, m, s, dtype, fast):
    ref64 = np.asarray(ref, dtype=np.float64)
    g = np.abs(np.log(ref64))
    if dtype == np.float32 and not fast:
        return ulp(ref, np.float32)
    rel = GAUSS_F32_FAST_REL * 2 if (fast and dtype == np.float32) else GAUSS_F64_REL * 2
    # exp turns an absolute error in g = m + s*z into a relative error in x
    return ref64 * rel * np.maximum(1.0, g) * max(1.0, s) + 4 * ulp(ref, dtype)


def check_close(got, ref, allowed, name=""):
    got64 = np.asarray(got, dtype=np.float64)
    ref64 = np.asarray(ref, dtype=np.float64)
    err = np.abs(got64 - ref64)
    bad = ~(err <= allowed)
    if bad.any():
        i = int(np.argmax(bad))
        raise AssertionError(
            f"{name}: {int(bad.sum())} of {len(err)} outside tolerance; first at {i}: got {got64[i]!r} "
            f"ref {ref64[i]!r} err {err[i]:.3e} allowed {allowed[i]:.3e}"
        )
    exact = float(np.mean(got64 == ref64)) if len(err) else 1.0
    return float(err.max()) if len(err) else 0.0, exact
