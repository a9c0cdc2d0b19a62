"""Stated tolerances for the floating-point distributions.

Test infrastructure (the checker side, like the rest of oracle/): only
tests/ and bench.py's per-rank slice check use it.

Integer words and uniform fp32/fp64 are compared bit-exactly elsewhere; the
functions here return the per-element allowed |gpu - ref| for gaussian and
lognormal outputs, given the reference (oracle) values.  Every bound is
written in fp32 ulps of the reference value or of the standard-normal
variate z (= (x - mean) / stddev), with the exhaustive measurements
(tools/bm_variants.cu, both 24-bit input grids, mean 0 / stddev 1) that back
it:

  gaussian fp32 "fast" (default): |err| <= 2^-20 * stddev * max(1, |z|)
      [measured worst 0.49 of it] and <= 8 ulp(z) for |z| >= 1 [6.7];
  gaussian fp32 "precise": <= 5 ulp(z) for every input [4.5];
  gaussian fp32 "accurate": the fp64 value cast once, <= 1 ulp;
  gaussian fp64: 2^-45 * stddev * max(1, |z|) (a few fp64 ulps);
  lognormal fp32 "fast": <= 10 ulp(x) * max(1, g) [8.2 worst over the
      dense-stream tests' parameter sets, 7.7 exhaustive at m = 0, s = 1],
  lognormal fp32 "precise": <= 6 ulp(x) * max(1, g) [5.1; 4.8 exhaustive],
      g = |m| + |ln x - m|: an fp32 exponent argument carries an error
      proportional to its magnitude, and exp turns that into a relative
      error of x (a condition number, not a method choice);
  lognormal fp32 "accurate": <= 1 ulp.
Each bound adds 2 ulp of the output and of mean / displ for the final
affine's own roundings when mean != 0 or stddev != 1.
"""

import numpy as np

GAUSS_F32_FAST_ABS = 2.0 ** -20  # x stddev x max(1, |z|)
GAUSS_F32_FAST_ULP_Z_GE_1 = 8.0
GAUSS_F32_PRECISE_ULP = 5.0
GAUSS_F64_REL = 2.0 ** -45
LOGN_F32_FAST_ULP = 10.0
LOGN_F32_PRECISE_ULP = 6.0


def ulp(x, dtype):
    x = np.abs(np.asarray(x, dtype=dtype))
    return np.spacing(x).astype(np.float64)


def ulp32(x):
    """fp32 ulp of x (x as fp64 values), normal range floor."""
    f = np.abs(np.asarray(x, dtype=np.float32)).astype(np.float64)
    f = np.maximum(f, np.finfo(np.float32).tiny)
    e = np.frexp(f)[1].astype(np.float64) - 1
    return np.ldexp(1.0, (e - 23).astype(np.int64))


def _method(fast):
    """fast may be a bool (True = "fast", False = "accurate") or a method name."""
    if fast is True:
        return "fast"
    if fast is False:
        return "accurate"
    return fast


def gaussian_allowed(ref, mean, stddev, dtype, fast):
    method = _method(fast)
    ref64 = np.asarray(ref, dtype=np.float64)
    z = (ref64 - mean) / stddev
    if dtype == np.float32 and method in ("accurate", "exact"):
        # accurate fp32 = fp64 math then one cast: at most 1 ulp from the cast
        return ulp(ref, np.float32)
    affine = 0.0 if (mean == 0.0 and stddev == 1.0) else 2 * ulp(ref, dtype) + 2 * ulp(mean, dtype)
    if dtype == np.float32 and method == "fast":
        a = stddev * GAUSS_F32_FAST_ABS * np.maximum(1.0, np.abs(z))
        return a + 2 * ulp(ref, dtype) + 2 * ulp(mean, dtype)
    if dtype == np.float32 and method == "precise":
        return GAUSS_F32_PRECISE_ULP * stddev * ulp32(z) + affine
    return stddev * GAUSS_F64_REL * np.maximum(1.0, np.abs(z)) + 2 * ulp(ref, dtype) + 2 * ulp(mean, dtype)


def gaussian_fast_ulp_claim(ref):
    """Standard normal (mean 0, stddev 1) "fast" outputs: the ulp part of the
    claim, <= 8 ulp where |z| >= 1 (elsewhere only the absolute bound)."""
    ref64 = np.asarray(ref, dtype=np.float64)
    return np.where(np.abs(ref64) >= 1.0, GAUSS_F32_FAST_ULP_Z_GE_1 * ulp32(ref64), np.inf)


def lognormal_allowed(ref, m, s, dtype, fast):
    method = _method(fast)
    ref64 = np.asarray(ref, dtype=np.float64)
    if dtype == np.float32 and method == "accurate":
        return ulp(ref, np.float32)
    with np.errstate(divide="ignore"):
        lx = np.log(np.maximum(ref64, np.finfo(np.float64).tiny))
    g = abs(m) + np.abs(lx - m)
    if dtype == np.float32 and method in ("fast", "precise"):
        k = LOGN_F32_FAST_ULP if method == "fast" else LOGN_F32_PRECISE_ULP
        return k * ulp32(ref64) * np.maximum(1.0, g)
    # fp64: exp turns an absolute error in g = m + s*z into a relative error in x
    return ref64 * GAUSS_F64_REL * 2 * np.maximum(1.0, g) * max(1.0, s) + 4 * ulp(ref, dtype)


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


def ulp_errors(got, ref):
    """|got - ref| in fp32 ulps of ref (for the band reports)."""
    return np.abs(np.asarray(got, dtype=np.float64) - np.asarray(ref, dtype=np.float64)) / ulp32(ref)
