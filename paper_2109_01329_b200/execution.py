"""CUDA task graph: the reference's buffer and USM submission styles on
streams, events and CUDA graphs.

Mirrors pkg/src/portarng/execution.py.  Buffers are device tensors in a
capped arena (execution.py:147-163); tasks are kernels over an element range
[start, stop) of their buffers, launched on the task's CUDA stream (the
current torch stream while the kernel callable runs).  Dependencies are
either inferred from buffer accessors -- read-after-write, write-after-read
and write-after-write, read_write counting as both (execution.py:222-272) --
or given as an explicit event list with no inference (execution.py:274-302),
exactly as in the reference.  Execution maps the DAG onto the GPU:

* ``Serial()``            -- one stream, tasks in submission order;
* ``Parallel(workers)``   -- a pool of ``workers`` streams; each splittable
  task is cut into the reference's chunks (execution.py:309-315) spread over
  the pool, every DAG edge becomes a CUDA event wait, independent tasks
  overlap;
* ``Graph(workers)``      -- the Parallel schedule captured once into a CUDA
  graph (cross-stream event edges become graph edges) and replayed.

Results are bitwise identical across backends for correctly declared graphs
(chunked generators regenerate from their stream offset); a missing USM edge
is a real race on the device, as with raw pointers.  Per-task start/end
times come from CUDA events on the task's streams.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple, Union

import enum

import numpy as np

from .distributions import Gaussian, Uniform, generate
from .engine import EngineState, _torch, skip_ahead
from .errors import Error

DEFAULT_ARENA_BYTES = 2 * 1024 ** 3  # execution.py:37
ARENA_ENV_VAR = "RNGBURN_ARENA_BYTES"  # execution.py:38

_KINDS = {"f32": ("float32", 4), "f64": ("float64", 8), "u32": ("uint32", 4)}

# Kernel callables receive the whole-buffer tensors and the element range
# [start, stop) they own; they launch on the current CUDA stream.
Kernel = Callable[[Dict[int, object], int, int], None]


class AllocationFailure(Error):
    """Arena cap exceeded or bad buffer spec (portarng.errors.AllocationFailure)."""


class UnknownBuffer(Error):
    """Buffer handle not owned by this graph, or listed twice (portarng.errors.UnknownBuffer)."""


class UnknownEvent(Error):
    """Event not owned by this graph (portarng.errors.UnknownEvent)."""


class KernelPanic(Error):
    """A task's kernel raised (portarng.errors.KernelPanic)."""


class PendingWrites(Error):
    """Host copy of a buffer an unexecuted task may still write (portarng.errors.PendingWrites)."""


class ConfigError(Error):
    """Malformed backend configuration (portarng.errors.ConfigError)."""


class AccessMode(enum.Enum):
    READ = "read"
    WRITE = "write"
    READ_WRITE = "read_write"


@dataclass(frozen=True)
class BufferHandle:
    id: int
    length: int
    kind: str


class Event:
    """Completion marker for one submitted task; completion is monotonic."""

    def __init__(self, task_id: int):
        self.task_id = task_id
        self._completed = False

    @property
    def completed(self) -> bool:
        return self._completed

    def _mark_complete(self) -> None:
        self._completed = True


@dataclass
class _Task:
    id: int
    fn: Kernel
    extent: int
    splittable: bool
    buffer_ids: Tuple[int, ...]
    writes: Tuple[int, ...]
    deps: Tuple[int, ...]
    executed: bool = False


@dataclass(frozen=True)
class Serial:
    pass


@dataclass(frozen=True)
class Parallel:
    workers: int
    chunk: Optional[int] = None

    def __post_init__(self):
        if self.workers < 1:
            raise ConfigError(f"parallel backend needs workers >= 1, got {self.workers}")
        if self.chunk is not None and self.chunk < 1:
            raise ConfigError(f"chunk must be positive, got {self.chunk}")


@dataclass(frozen=True)
class Graph(Parallel):
    """Parallel schedule captured into one CUDA graph, then replayed."""


Backend = Union[Serial, Parallel, Graph]


def parse_backend(text: str) -> Backend:
    """'serial', 'parallel:N' or 'graph:N' (execution.py:107-117 plus graph)."""
    if text == "serial":
        return Serial()
    for prefix, cls in (("parallel:", Parallel), ("graph:", Graph)):
        if text.startswith(prefix):
            try:
                return cls(workers=int(text.split(":", 1)[1]))
            except ValueError as exc:
                raise ConfigError(f"bad backend spec {text!r}") from exc
    raise ConfigError(f"backend must be serial, parallel:N or graph:N, got {text!r}")


def backend_label(backend: Backend) -> str:
    if isinstance(backend, Serial):
        return "serial"
    return f"{'graph' if isinstance(backend, Graph) else 'parallel'}:{backend.workers}"


@dataclass
class TaskReport:
    task_id: int
    start_ns: int
    end_ns: int

    @property
    def duration_ns(self) -> int:
        return self.end_ns - self.start_ns


@dataclass
class RunReport:
    tasks: List[TaskReport] = field(default_factory=list)
    total_ns: int = 0


class TaskGraph:
    """Device buffers plus submitted tasks and their dependency edges (always acyclic)."""

    def __init__(self, arena_bytes: Optional[int] = None, device="cuda"):
        if arena_bytes is None:
            arena_bytes = int(os.environ.get(ARENA_ENV_VAR, DEFAULT_ARENA_BYTES))
        self.arena_bytes = arena_bytes
        self.allocated_bytes = 0
        self.device = device
        self._storage: Dict[int, object] = {}
        self._handles: Dict[int, BufferHandle] = {}
        self._tasks: List[_Task] = []
        self._events: Dict[int, Event] = {}
        self.edges: set = set()
        self._last_writer: Dict[int, int] = {}
        self._readers_since_write: Dict[int, List[int]] = {}
        self.transfer_ns = 0
        self._graph_cache = None

    # -- buffers ------------------------------------------------------------

    def create_buffer(self, n: int, kind: str = "f32") -> BufferHandle:
        """Allocate a zero-initialised device buffer of n elements (execution.py:147-163)."""
        if n < 0:
            raise AllocationFailure("buffer length must be non-negative")
        if kind not in _KINDS:
            raise AllocationFailure(f"unknown element kind {kind!r}")
        nbytes = n * _KINDS[kind][1]
        if self.allocated_bytes + nbytes > self.arena_bytes:
            raise AllocationFailure(f"arena cap exceeded: {self.allocated_bytes + nbytes} > {self.arena_bytes} bytes")
        torch = _torch()
        handle = BufferHandle(id=len(self._handles), length=n, kind=kind)
        self._storage[handle.id] = torch.zeros(n, dtype=getattr(torch, _KINDS[kind][0]), device=self.device)
        self._handles[handle.id] = handle
        self.allocated_bytes += nbytes
        self._readers_since_write[handle.id] = []
        return handle

    def _check_handle(self, handle: BufferHandle) -> None:
        if self._handles.get(handle.id) is not handle:
            raise UnknownBuffer(f"buffer {handle!r} does not belong to this graph")

    def buffer_view(self, handle: BufferHandle):
        """The buffer's device tensor."""
        self._check_handle(handle)
        return self._storage[handle.id]

    # -- submission ---------------------------------------------------------

    def _add_task(self, fn: Kernel, buffer_ids, writes, deps, extent, splittable) -> Event:
        if extent is None:
            extent = max((self._handles[b].length for b in buffer_ids), default=0)
        task = _Task(id=len(self._tasks), fn=fn, extent=extent, splittable=splittable,
                     buffer_ids=tuple(buffer_ids), writes=tuple(writes), deps=tuple(sorted(set(deps))))
        self._tasks.append(task)
        for dep in task.deps:
            self.edges.add((dep, task.id))
        assert all(u < v for u, v in self.edges), "dependency edge points backwards"
        event = Event(task.id)
        self._events[task.id] = event
        self._graph_cache = None
        return event

    def submit_with_accessors(self, kernel: Kernel, accessors: Sequence[Tuple[BufferHandle, AccessMode]],
                              extent: Optional[int] = None, splittable: bool = True) -> Event:
        """Dependencies inferred from access modes (execution.py:222-272): readers
        depend on the last writer (RAW); a writer depends on every reader since
        the last write (WAR) and on the last writer (WAW)."""
        seen = set()
        for handle, mode in accessors:
            self._check_handle(handle)
            if handle.id in seen:
                raise UnknownBuffer(f"buffer {handle.id} listed twice in one task")
            seen.add(handle.id)
            if not isinstance(mode, AccessMode):
                raise ConfigError(f"bad access mode {mode!r}")
        deps: List[int] = []
        writes: List[int] = []
        for handle, mode in accessors:
            reads_buf = mode in (AccessMode.READ, AccessMode.READ_WRITE)
            writes_buf = mode in (AccessMode.WRITE, AccessMode.READ_WRITE)
            if reads_buf and handle.id in self._last_writer:
                deps.append(self._last_writer[handle.id])
            if writes_buf:
                deps.extend(self._readers_since_write[handle.id])
                if handle.id in self._last_writer:
                    deps.append(self._last_writer[handle.id])
                writes.append(handle.id)
        event = self._add_task(kernel, [h.id for h, _ in accessors], writes, deps, extent, splittable)
        for handle, mode in accessors:
            if mode in (AccessMode.WRITE, AccessMode.READ_WRITE):
                self._last_writer[handle.id] = event.task_id
                self._readers_since_write[handle.id] = []
            if mode in (AccessMode.READ, AccessMode.READ_WRITE):
                self._readers_since_write[handle.id].append(event.task_id)
        return event

    def submit_with_events(self, kernel: Kernel, buffers_unchecked: Sequence[BufferHandle], deps: Sequence[Event],
                           extent: Optional[int] = None, splittable: bool = True) -> Event:
        """Ordered only by the given events; nothing inferred (execution.py:274-302).
        A missing real dependency is the caller's race, as with raw pointers."""
        for handle in buffers_unchecked:
            self._check_handle(handle)
        for ev in deps:
            if self._events.get(ev.task_id) is not ev:
                raise UnknownEvent(f"event for task {ev.task_id} does not belong to this graph")
        ids = [h.id for h in buffers_unchecked]
        return self._add_task(kernel, ids, ids, [ev.task_id for ev in deps], extent, splittable)

    # -- execution ----------------------------------------------------------

    def _views(self, task: _Task) -> Dict[int, object]:
        return {b: self._storage[b] for b in task.buffer_ids}

    @staticmethod
    def _chunks(task: _Task, backend: Backend) -> List[Tuple[int, int]]:
        """execution.py:309-315."""
        if isinstance(backend, Serial) or not task.splittable or task.extent == 0:
            return [(0, task.extent)]
        size = backend.chunk
        if size is None:
            size = max(4096, -(-task.extent // (4 * backend.workers)))
        return [(a, min(a + size, task.extent)) for a in range(0, task.extent, size)]

    def _issue(self, pending: List[_Task], backend: Backend, streams, timing: bool):
        """Launch every pending task on the stream pool in submission order
        (a topological order: edges point forward).  Each task waits on the
        end events of its pending predecessors; its chunks go round-robin
        over the pool.  Returns {task id: ([start events], [end events])}."""
        torch = _torch()
        done_ev: Dict[int, List[object]] = {}
        marks: Dict[int, Tuple[list, list]] = {}
        rr = 0
        ext = isinstance(backend, Graph)
        for task in pending:
            chunks = self._chunks(task, backend)
            views = self._views(task)
            starts, ends, deps = [], [], []
            for ci, (a, b) in enumerate(chunks):
                s = streams[0] if isinstance(backend, Serial) else streams[(rr + ci) % len(streams)]
                for d in task.deps:
                    for e in done_ev.get(d, ()):
                        s.wait_event(e)
                with torch.cuda.stream(s):
                    if timing:  # inside a capture: event-record nodes (external)
                        st = torch.cuda.Event(enable_timing=True, external=ext)
                        st.record(s)
                        starts.append(st)
                    try:
                        task.fn(views, a, b)
                    except Exception as exc:
                        raise KernelPanic(f"task {task.id} failed: {exc}") from exc
                    if timing:
                        en = torch.cuda.Event(enable_timing=True, external=ext)
                        en.record(s)
                        ends.append(en)
                    if ext or not timing:  # dependency marker (a graph edge when captured)
                        dep = torch.cuda.Event()
                        dep.record(s)
                        deps.append(dep)
                    else:
                        deps.append(en)
            rr += len(chunks)
            done_ev[task.id] = deps
            marks[task.id] = (starts, ends)
        return marks

    def run(self, backend: Backend) -> RunReport:
        """Execute all pending tasks; predecessors always finish first
        (execution.py:317-341).  Blocks until the device is done."""
        if not isinstance(backend, (Serial, Parallel)):
            raise ConfigError(f"unknown backend {backend!r}")
        torch = _torch()
        pending = [t for t in self._tasks if not t.executed]
        report = RunReport()
        if not pending:
            return report
        dev = torch.device(self.device)
        if dev.type != "cuda":
            raise ConfigError("TaskGraph.run executes on a CUDA device")
        nstreams = 1 if isinstance(backend, Serial) else backend.workers
        base_stream = torch.cuda.current_stream(dev)
        streams = [torch.cuda.Stream(dev) for _ in range(nstreams)]
        t_run0 = time.perf_counter_ns()
        origin = torch.cuda.Event(enable_timing=True)
        origin.record(base_stream)
        for s in streams:
            s.wait_stream(base_stream)
        if isinstance(backend, Graph):
            marks = self._run_graph(pending, backend, streams, base_stream, dev)
        else:
            marks = self._issue(pending, backend, streams, timing=True)
        for s in streams:
            base_stream.wait_stream(s)
        base_stream.synchronize()
        report.total_ns = time.perf_counter_ns() - t_run0
        for task in pending:
            starts, ends = marks[task.id]
            t0 = min(origin.elapsed_time(e) for e in starts) if starts else 0.0
            t1 = max(origin.elapsed_time(e) for e in ends) if ends and starts else t0
            report.tasks.append(TaskReport(task.id, t_run0 + int(t0 * 1e6), t_run0 + int(t1 * 1e6)))
            task.executed = True
            self._events[task.id]._mark_complete()
        return report

    def _run_graph(self, pending, backend, streams, base_stream, dev):
        """Capture the Parallel schedule once (stream 0 forks to the pool
        through events, so every DAG edge is a graph edge) and replay it."""
        torch = _torch()
        key = (tuple(t.id for t in pending), backend)
        if self._graph_cache is None or self._graph_cache[0] != key:
            g = torch.cuda.CUDAGraph()
            cap = streams[0]
            with torch.cuda.graph(g, stream=cap):
                fork = torch.cuda.Event()
                fork.record(cap)
                for s in streams[1:]:
                    s.wait_event(fork)
                marks = self._issue(pending, backend, streams, timing=True)
                for s in streams[1:]:
                    cap.wait_stream(s)
            self._graph_cache = (key, g, marks)
        _, g, marks = self._graph_cache
        with torch.cuda.stream(streams[0]):
            g.replay()
        return marks

    # -- host transfer ------------------------------------------------------

    def copy_to_host(self, handle: BufferHandle) -> np.ndarray:
        """Snapshot a device buffer into host memory; the copy time is recorded
        (execution.py:428-442).  PendingWrites while an unexecuted task may
        still write it (event-list tasks count as writers of every buffer
        they list)."""
        self._check_handle(handle)
        for task in self._tasks:
            if not task.executed and handle.id in task.writes:
                raise PendingWrites(f"buffer {handle.id} has pending writer task {task.id}")
        t0 = time.perf_counter_ns()
        host = self._storage[handle.id].cpu().numpy()
        self.transfer_ns += time.perf_counter_ns() - t0
        return host


# ---------------------------------------------------------------- device kernels
# The reference burner's kernels (rngburn.py:62-100) as chunkable device
# launches: a chunk regenerates from its own stream offset, so any split is
# bitwise identical to one launch.


def uniform_generate_kernel(base_state: EngineState, buf_id: int, precision: str) -> Kernel:
    """rngburn.py:67-75: unit uniforms; chunk [start, stop) = stream words start.. ."""
    spec = Uniform(0.0, 1.0, precision)

    def kernel(views, start, stop):
        if stop > start:
            state = base_state if start == 0 else skip_ahead(base_state, start)
            generate(spec, state, stop - start, out=views[buf_id][start:stop])

    return kernel


def gaussian_generate_kernel(base_state: EngineState, buf_id: int, mean: float, stddev: float,
                             precision: str, method: str = "fast") -> Kernel:
    """rngburn.py:78-91: normals; pair k uses stream words 2k, 2k+1, so a chunk
    starting at an odd element regenerates its first pair and drops the cosine."""
    spec = Gaussian(mean, stddev, precision, method)

    def kernel(views, start, stop):
        if stop <= start:
            return
        out = views[buf_id]
        if start % 2 == 0:
            state = base_state if start == 0 else skip_ahead(base_state, start)
            generate(spec, state, stop - start, out=out[start:stop])
            return
        first_pair = start // 2
        state = skip_ahead(base_state, 2 * first_pair)
        _, tmp = generate(spec, state, stop - 2 * first_pair,
                          out=_torch().empty(stop - 2 * first_pair, dtype=out.dtype, device=out.device))
        out[start:stop].copy_(tmp[1:])

    return kernel


def affine_kernel(buf_id: int, lo: float, hi: float) -> Kernel:
    """rngburn.py:94-100 / 62-64: in-place v *= (hi - lo); v += lo (two roundings)."""
    from . import _lib
    from .engine import _stream_handle

    def kernel(views, start, stop):
        v = views[buf_id]
        if stop <= start:
            return
        fn = _lib.lib.prng_range_transform_f32 if v.element_size() == 4 else _lib.lib.prng_range_transform_f64
        seg = v[start:stop]
        _lib.check(fn(seg.data_ptr(), stop - start, lo, hi, _stream_handle(None, v.device)))

    return kernel
