"""RNG burner on the GPU: timed generate ->
transform -> copy-back cycles with the reference's result format.

Mirrors pkg/src/portarng/rngburn.py: `burn_once` is one time-to-solution
cycle as the paper defines it (construction, allocation,
generation, range transform, synchronisation, device-to-host copy), the API
modes keep the reference's names, and results are written in its exact CSV
schema (rngburn.py:34, 183-192) so `portarng.rngburn.compare` can compute
slowdowns and P between a GPU file and a CPU file.

API modes on CUDA (rngburn.py:127-149), through the CUDA task graph
(execution.py in this package):
* ``"buffer"``  -- generate and range-transform tasks submitted with
  read_write accessors; the inferred RAW edge orders them;
* ``"usm"``     -- the same two tasks with an explicit event dependency;
* ``"hostdirect"`` -- the fused single-kernel library call (the native-baseline
  role), then the identity transform for gaussians as the reference applies it.
The backend (Serial / Parallel(workers) / Graph(workers)) maps the graph onto
one stream, a stream pool, or a replayed CUDA graph.  All combinations
produce bit-identical output (tests/test_burner.py).
"""

from __future__ import annotations

import csv
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

from . import _lib
from .distributions import Gaussian, Uniform, generate
from .engine import EngineKind, _stream_handle, _torch, seed_engine
from .errors import Error, InvalidParameter
from .execution import (AccessMode, Backend, ConfigError, Serial, TaskGraph, affine_kernel, backend_label,
                        gaussian_generate_kernel, uniform_generate_kernel)

CSV_HEADER = ["platform", "api", "backend", "engine", "dist", "batch", "iter", "tts_ns"]  # rngburn.py:34
API_MODES = ("buffer", "usm", "hostdirect")


class SchemaMismatch(Error):
    """CSV file does not carry the expected header (portarng.errors.SchemaMismatch)."""


def dist_label(spec) -> str:
    """distributions.py:156-160."""
    if isinstance(spec, Uniform):
        return f"uniform:{spec.lo:g}:{spec.hi:g}"
    return f"gaussian:{spec.mean:g}:{spec.stddev:g}"


@dataclass
class RunRecord:
    """metrics.py:23-39 (same fields)."""

    platform: str
    api_mode: str
    backend: str
    engine: str
    dist: str
    batch: int
    samples: List[int] = field(default_factory=list)


@dataclass
class BurnConfig:
    """rngburn.py:41-59 (backend = a CUDA task-graph backend)."""

    engine: EngineKind
    dist: object
    api_mode: str
    backend: Backend
    batches: List[int]
    iterations: int = 100
    seed: int = 0
    out_path: Optional[str] = None
    platform: str = "b200"
    device: str = "cuda:0"

    def __post_init__(self):
        if self.api_mode not in API_MODES:
            raise ConfigError(f"api mode must be one of {API_MODES}, got {self.api_mode!r}")
        if not self.batches or any(b < 1 for b in self.batches):
            raise ConfigError(f"batch sizes must be >= 1, got {self.batches}")
        if self.iterations < 1:
            raise ConfigError(f"iterations must be >= 1, got {self.iterations}")


def _transform_range(spec) -> Tuple[float, float]:
    # rngburn.py:103-108: gaussian batches keep an identity transform
    return (spec.lo, spec.hi) if isinstance(spec, Uniform) else (0.0, 1.0)


def burn_once(engine: EngineKind, spec, api_mode: str, backend: Backend, batch: int, seed: int,
              device: str = "cuda:0") -> Tuple[int, object]:
    """One timed full cycle on the GPU; returns (tts_ns, host numpy array).  rngburn.py:111-151."""
    torch = _torch()
    if api_mode not in API_MODES:
        raise ConfigError(f"api mode must be one of {API_MODES}, got {api_mode!r}")
    if not isinstance(spec, (Uniform, Gaussian)):
        raise InvalidParameter("the burner runs uniform or gaussian requests")
    lo, hi = _transform_range(spec)
    precision = spec.precision
    dev = torch.device(device)
    t0 = time.perf_counter_ns()
    state = seed_engine(engine, seed)
    if api_mode == "hostdirect":
        s0 = torch.cuda.current_stream(dev)
        buf = torch.empty(batch, dtype=torch.float32 if precision == "fp32" else torch.float64, device=dev)
        generate(spec, state, batch, out=buf, stream=s0)
        if isinstance(spec, Gaussian):  # identity transform, as the reference applies it
            fn = _lib.lib.prng_range_transform_f32 if precision == "fp32" else _lib.lib.prng_range_transform_f64
            _lib.check(fn(buf.data_ptr(), batch, lo, hi, _stream_handle(s0)))
        host = buf.cpu().numpy()
    else:
        graph = TaskGraph(arena_bytes=max(2 * 1024 ** 3, 8 * batch), device=dev)
        buf = graph.create_buffer(batch, "f32" if precision == "fp32" else "f64")
        if isinstance(spec, Uniform):
            gen = uniform_generate_kernel(state, buf.id, precision)
        else:
            gen = gaussian_generate_kernel(state, buf.id, spec.mean, spec.stddev, precision, spec.method)
        tr = affine_kernel(buf.id, lo, hi)
        if api_mode == "buffer":
            graph.submit_with_accessors(gen, [(buf, AccessMode.READ_WRITE)])
            graph.submit_with_accessors(tr, [(buf, AccessMode.READ_WRITE)])
        else:  # usm
            e1 = graph.submit_with_events(gen, [buf], deps=[])
            graph.submit_with_events(tr, [buf], deps=[e1])
        graph.run(backend)
        host = graph.copy_to_host(buf)
    tts = time.perf_counter_ns() - t0
    return tts, host


def run_burner(config: BurnConfig) -> List[RunRecord]:
    """rngburn.py:154-177: every batch size, `iterations` cycles each."""
    records = []
    for batch in config.batches:
        samples = []
        for _ in range(config.iterations):
            tts, _ = burn_once(config.engine, config.dist, config.api_mode, config.backend, batch, config.seed,
                               config.device)
            samples.append(tts)
        records.append(RunRecord(config.platform, config.api_mode, backend_label(config.backend),
                                 config.engine.value, dist_label(config.dist), batch, samples))
    if config.out_path:
        write_records_csv(records, config.out_path)
    return records


def write_records_csv(records: Sequence[RunRecord], path: str) -> None:
    """Byte-compatible with rngburn.write_records_csv (rngburn.py:183-192)."""
    with open(path, "w", newline="") as f:
        writer = csv.writer(f, lineterminator="\n")
        writer.writerow(CSV_HEADER)
        for rec in records:
            for it, tts in enumerate(rec.samples):
                writer.writerow([rec.platform, rec.api_mode, rec.backend, rec.engine, rec.dist, rec.batch, it, tts])


def read_rows_csv(path: str) -> List[dict]:
    """rngburn.read_rows_csv (rngburn.py:195-217): exact header enforced."""
    with open(path, newline="") as f:
        reader = csv.reader(f)
        header = next(reader, None)
        if header != CSV_HEADER:
            raise SchemaMismatch(f"{path}: expected header {CSV_HEADER}, got {header}")
        rows = []
        for row in reader:
            if len(row) != len(CSV_HEADER):
                raise SchemaMismatch(f"{path}: malformed row {row!r}")
            rows.append({"platform": row[0], "api": row[1], "backend": row[2], "engine": row[3], "dist": row[4],
                         "batch": int(row[5]), "iter": int(row[6]), "tts_ns": int(row[7])})
    return rows
