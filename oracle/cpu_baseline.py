"""CPU baseline of the hot path -- bench.py's cpu_baseline / --impl reference leg.

TEST/BENCH INFRASTRUCTURE ONLY (see oracle/oracle.py header).

Restates the reference's own multi-core path for one burner cycle,
burn_once(engine, Uniform, "buffer", Parallel(workers), n, seed)
(rngburn.py:111-151, execution.py:309-424): the element range is cut into
chunks of max(4096, ceil(n / (4 * workers))) (execution.py:314), each chunk
regenerates its words from skip_ahead(base, start) with the reference's
compiled kernel core (_core.philox_fill, nogil -> truly parallel threads,
_core.pyx:55), maps them with words_to_unit (distributions.py:83-87) into the
output buffer, and a second pass applies the affine range transform
(rngburn.py:94-100).  MRG32k3a is unsplittable in the reference
(rngburn.py:123) and runs as one chunk.

kind = "reference" when the reference core built into oracle/_ref is
importable; otherwise the plain-C restatement (oracle.c) stands in with
kind = "port".
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import oracle as O


class CpuPath:
    def __init__(self, workers: int | None = None):
        self.core = O.ref_core()
        self.kind = "reference" if self.core is not None else "port"
        self.workers = workers or os.cpu_count() or 1
        self.pool = ThreadPoolExecutor(max_workers=self.workers)

    def _philox_fill(self, key, pos, n):
        block, lane = divmod(pos, 4)
        b = [(block >> (32 * i)) & 0xFFFFFFFF for i in range(4)]
        if self.core is not None:
            return self.core.philox_fill(key[0], key[1], *b, lane, n)
        return O.philox_fill(key[0], key[1], *b, lane, n)

    def _mrg_fill(self, s1, s2, n):
        if self.core is not None:
            return self.core.mrg_fill(*s1, *s2, n)[0]
        return O.mrg_fill(*s1, *s2, n)[0]

    def burn_philox_uniform(self, key, pos, n, lo=0.0, hi=1.0, precision="fp32", out=None):
        """One generate -> transform cycle into `out` (allocated if None)."""
        dtype = np.float32 if precision == "fp32" else np.float64
        if out is None:
            out = np.empty(n, dtype=dtype)
        chunk = max(4096, -(-n // (4 * self.workers)))

        def gen(start):
            stop = min(n, start + chunk)
            w = self._philox_fill(key, pos + start, stop - start)
            out[start:stop] = O.words_to_unit(w, precision)

        def affine(start):
            O.range_transform(out[start:min(n, start + chunk)], lo, hi)

        list(self.pool.map(gen, range(0, n, chunk)))
        list(self.pool.map(affine, range(0, n, chunk)))
        return out

    def burn_mrg_uniform(self, s1, s2, n, lo=0.0, hi=1.0, precision="fp64"):
        w = self._mrg_fill(s1, s2, n)
        return O.range_transform(O.words_to_unit(w, precision), lo, hi)

    def _box_muller(self, u1, u2):
        if self.core is not None:
            return self.core.box_muller(u1, u2)
        return O.box_muller(u1, u2)

    def burn_philox_gaussian(self, key, pos, n, mean=0.0, stddev=1.0, precision="fp32", out=None):
        """One gaussian cycle like rngburn.gaussian_generate_kernel chunks
        (rngburn.py:78-91): each even-aligned chunk draws its words, the core's
        box_muller (_core.pyx:105-122) on (1 - u1, u2), x stddev + mean in
        fp64, cast (distributions.py:116-131)."""
        dtype = np.float32 if precision == "fp32" else np.float64
        if out is None:
            out = np.empty(n, dtype=dtype)
        chunk = max(4096, -(-n // (4 * self.workers)))
        chunk += chunk & 1

        def gen(start):
            stop = min(n, start + chunk)
            m = stop - start
            w = self._philox_fill(key, pos + start, m + (m & 1))
            u1 = (w[0::2] >> np.uint32(8)).astype(np.float64) * O.UNIT_SCALE
            u2 = (w[1::2] >> np.uint32(8)).astype(np.float64) * O.UNIT_SCALE
            z0, z1 = self._box_muller(1.0 - u1, u2)
            z = np.empty(2 * len(u1), dtype=np.float64)
            z[0::2] = z0
            z[1::2] = z1
            z *= stddev
            z += mean
            out[start:stop] = z[:m]

        list(self.pool.map(gen, range(0, n, chunk)))
        return out

    def time_cycle(self, fn, reps=3):
        """Best-of-reps seconds of fn()."""
        best = float("inf")
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            best = min(best, time.perf_counter() - t0)
        return best

    def time_philox_uniform(self, n, reps=3, key=(777, 0), pos=0):
        """Best-of-reps seconds for one cycle of n fp32 uniforms (plus the output)."""
        out = np.empty(n, dtype=np.float32)
        best = float("inf")
        for _ in range(reps):
            t0 = time.perf_counter()
            self.burn_philox_uniform(key, pos, n, out=out)
            best = min(best, time.perf_counter() - t0)
        return best, out

    def close(self):
        self.pool.shutdown()
