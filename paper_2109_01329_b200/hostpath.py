"""Generate straight into host memory (the paper's TTS shape: generate,
transform, copy back, rngburn.py:125-150).

Two strategies, both a single pass over HBM or none at all:

* ``"zero_copy"`` -- the fused kernel's stores target mapped pinned host
  memory directly (the C ABI accepts a pinned host pointer as `out`), so
  samples cross PCIe / C2C exactly once and never touch HBM;
* ``"pipelined"`` -- chunks are generated into two device staging buffers on
  two streams while the previous chunk is copied device -> host, so
  generation hides under the copy.
"""

from __future__ import annotations

from .distributions import DistributionSpec, Gaussian, Lognormal, generate, out_dtype, words_consumed
from .engine import EngineState, Mrg32k3a, Philox4x32x10, _torch, skip_ahead
from .errors import InvalidParameter

_CHUNK = 1 << 25


class HostGenerator:
    """Reusable staging state for repeated host-buffer requests on one device."""

    def __init__(self, device=None, chunk: int = _CHUNK, strategy: str = "pipelined"):
        torch = _torch()
        if strategy not in ("pipelined", "zero_copy"):
            raise InvalidParameter(f"unknown strategy {strategy!r}")
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.chunk = chunk
        self.strategy = strategy
        self.streams = [torch.cuda.Stream(self.device), torch.cuda.Stream(self.device)]
        self._bufs = {}

    def _buffers(self, dtype):
        torch = _torch()
        if dtype not in self._bufs:
            self._bufs[dtype] = [torch.empty(self.chunk, dtype=dtype, device=self.device) for _ in range(2)]
        return self._bufs[dtype]

    def generate(self, spec: DistributionSpec, state: EngineState, n: int, host_out):
        """Fill host_out[:n] (pinned CPU tensor); returns the advanced state
        (a stateful Philox4x32x10 / Mrg32k3a engine is advanced in place and
        returned).  Work is enqueued on this generator's streams; call
        synchronize()."""
        torch = _torch()
        if host_out.is_cuda or not host_out.is_pinned():
            raise InvalidParameter("host_out must be a pinned CPU tensor")
        if n < 0:
            raise InvalidParameter("count must be non-negative")
        if isinstance(state, (Philox4x32x10, Mrg32k3a)):
            # validate and enqueue on the immutable state first; advance the
            # engine object only once every chunk is enqueued
            engine = state
            self.generate(spec, engine.state, n, host_out)
            return engine.skip_ahead(words_consumed(spec, n))
        if self.strategy == "zero_copy":
            s = self.streams[0]
            generate(spec, state, n, out=host_out, stream=s)
            return skip_ahead(state, words_consumed(spec, n)) if n else state
        pair = isinstance(spec, (Gaussian, Lognormal))
        chunk = self.chunk - (self.chunk % 2 if pair else 0)
        bufs = self._buffers(out_dtype(spec))
        cur = state
        for i, start in enumerate(range(0, n, chunk)):
            m = min(chunk, n - start)
            s = self.streams[i % 2]
            with torch.cuda.stream(s):
                generate(spec, cur, m, out=bufs[i % 2], stream=s)
                host_out[start:start + m].copy_(bufs[i % 2][:m], non_blocking=True)
            cur = skip_ahead(cur, words_consumed(spec, m))
        return cur

    def synchronize(self):
        for s in self.streams:
            s.synchronize()
