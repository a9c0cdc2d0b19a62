"""CUDA task graph (execution.py analogue) -- the reference's
tests/test_execution.py behaviours: accessor hazard edges, event-list
submission, arena cap, pending writes on CPU (host bookkeeping only, device
"meta"), and on the GPU: serial == chunked multi-stream == CUDA graph
bitwise, topological start order from device timestamps, the USM race with a
missing edge, kernel panics, generate->transform chains equal to the oracle."""

import numpy as np
import pytest

import paper_2109_01329_b200 as P
from paper_2109_01329_b200 import execution as X

R, W, RW = X.AccessMode.READ, X.AccessMode.WRITE, X.AccessMode.READ_WRITE


def fill_kernel(buf_id, value):
    def kernel(views, start, stop):
        views[buf_id][start:stop] = value

    return kernel


def add_kernel(dst_id, src_id, scale=1.0):
    def kernel(views, start, stop):
        views[dst_id][start:stop] += views[src_id][start:stop] * scale

    return kernel


def scale_kernel(buf_id, factor):
    def kernel(views, start, stop):
        views[buf_id][start:stop] *= factor

    return kernel


def meta_graph(**kw):
    return X.TaskGraph(device="meta", **kw)


# ------------------------------------------------------------ host bookkeeping


def test_create_buffer_ids_and_arena_cap(monkeypatch):
    g = meta_graph()
    a, b = g.create_buffer(0), g.create_buffer(8)
    assert a.length == 0 and a.id != b.id
    small = meta_graph(arena_bytes=256 * 1024 * 1024)
    with pytest.raises(X.AllocationFailure):
        small.create_buffer(10 ** 8, "f32")
    meta_graph(arena_bytes=2 * 1024 ** 3).create_buffer(10 ** 8, "f32")
    with pytest.raises(X.AllocationFailure):
        g.create_buffer(4, "f16")
    with pytest.raises(X.AllocationFailure):
        g.create_buffer(-1)
    monkeypatch.setenv("RNGBURN_ARENA_BYTES", "1024")
    g = meta_graph()
    assert g.arena_bytes == 1024
    with pytest.raises(X.AllocationFailure):
        g.create_buffer(1024, "f32")


def test_unknown_and_duplicate_buffers_rejected():
    g1, g2 = meta_graph(), meta_graph()
    foreign = g2.create_buffer(4)
    with pytest.raises(X.UnknownBuffer):
        g1.submit_with_accessors(fill_kernel(foreign.id, 1.0), [(foreign, W)])
    a = g1.create_buffer(4)
    with pytest.raises(X.UnknownBuffer):
        g1.submit_with_accessors(fill_kernel(a.id, 1.0), [(a, R), (a, W)])


def test_hazard_edges():
    g = meta_graph()
    a, b, out = g.create_buffer(8), g.create_buffer(8), g.create_buffer(8)
    e1 = g.submit_with_accessors(fill_kernel(a.id, 0.5), [(a, RW)])
    e2 = g.submit_with_accessors(scale_kernel(a.id, 2.0), [(a, RW)])
    assert (e1.task_id, e2.task_id) in g.edges  # RAW generate -> transform
    g.submit_with_accessors(fill_kernel(b.id, 2.0), [(b, W)])
    assert len(g.edges) == 1  # disjoint writers: no edge
    w0 = g.submit_with_accessors(fill_kernel(a.id, 1.0), [(a, W)])
    r1 = g.submit_with_accessors(add_kernel(out.id, a.id), [(out, RW), (a, R)])
    w2 = g.submit_with_accessors(fill_kernel(a.id, 3.0), [(a, W)])
    assert (w0.task_id, r1.task_id) in g.edges  # RAW
    assert (r1.task_id, w2.task_id) in g.edges  # WAR
    assert (w0.task_id, w2.task_id) in g.edges  # WAW
    assert all(u < v for u, v in g.edges)


def test_read_write_chain_is_linear():
    g = meta_graph()
    a = g.create_buffer(8)
    ids = [g.submit_with_accessors(scale_kernel(a.id, 2.0), [(a, RW)]).task_id for _ in range(3)]
    assert (ids[0], ids[1]) in g.edges and (ids[1], ids[2]) in g.edges
    assert (ids[0], ids[2]) not in g.edges


def test_event_edges_and_foreign_event():
    g1, g2 = meta_graph(), meta_graph()
    a = g1.create_buffer(8)
    e1 = g1.submit_with_events(fill_kernel(a.id, 1.0), [a], deps=[])
    e2 = g1.submit_with_events(scale_kernel(a.id, 2.0), [a], deps=[e1])
    assert (e1.task_id, e2.task_id) in g1.edges
    b = g2.create_buffer(4)
    ev = g2.submit_with_events(fill_kernel(b.id, 1.0), [b], deps=[])
    with pytest.raises(X.UnknownEvent):
        g1.submit_with_events(fill_kernel(a.id, 1.0), [a], deps=[ev])


def test_pending_writes_and_backend_parsing():
    g = meta_graph()
    a = g.create_buffer(16)
    g.submit_with_accessors(fill_kernel(a.id, 1.0), [(a, W)])
    with pytest.raises(X.PendingWrites):
        g.copy_to_host(a)
    assert X.parse_backend("serial") == X.Serial()
    assert X.parse_backend("parallel:8") == X.Parallel(8)
    assert X.parse_backend("graph:4") == X.Graph(4)
    assert X.backend_label(X.Parallel(3)) == "parallel:3" and X.backend_label(X.Graph(2)) == "graph:2"
    for bad in ("gpu", "parallel:x"):
        with pytest.raises(X.ConfigError):
            X.parse_backend(bad)
    with pytest.raises(X.ConfigError):
        X.Parallel(0)
    assert X.TaskGraph._chunks(X._Task(0, None, 100003, True, (), (), ()), X.Parallel(4)) == \
        [(a, min(a + 6251, 100003)) for a in range(0, 100003, 6251)]  # max(4096, ceil(n / 16))


# ------------------------------------------------------------------- on the GPU

torch = pytest.importorskip("torch")
gpu = pytest.mark.skipif(not torch.cuda.is_available(), reason="no CUDA device")
BACKENDS = (X.Serial(), X.Parallel(2, chunk=9973), X.Parallel(4), X.Graph(3, chunk=3331), X.Graph(8))


@pytest.mark.gpu
@gpu
def test_event_chain_runs_in_order_and_completes():
    g = X.TaskGraph()
    a = g.create_buffer(8)
    e1 = g.submit_with_events(fill_kernel(a.id, 1.0), [a], deps=[])
    g.submit_with_events(scale_kernel(a.id, 2.0), [a], deps=[e1])
    assert not e1.completed
    g.run(X.Serial())
    assert e1.completed and np.all(g.copy_to_host(a) == 2.0)
    g.submit_with_accessors(scale_kernel(a.id, 2.0), [(a, RW)])
    g.run(X.Parallel(2))
    assert e1.completed and np.all(g.copy_to_host(a) == 4.0)
    assert X.TaskGraph().run(X.Serial()).tasks == []


@pytest.mark.gpu
@gpu
def test_missing_usm_dependency_is_a_device_race():
    def build(with_dep, delay):
        g = X.TaskGraph()
        a = g.create_buffer(64)

        def slow_fill(views, start, stop):
            if delay:
                torch.cuda._sleep(100_000_000)  # ~50 ms of device time before the write
            views[a.id][start:stop] = 1.0

        e1 = g.submit_with_events(slow_fill, [a], deps=[], splittable=False)
        g.submit_with_events(scale_kernel(a.id, 2.0), [a], deps=[e1] if with_dep else [], splittable=False)
        return g, a

    g, a = build(True, False)
    g.run(X.Serial())
    oracle = g.copy_to_host(a)
    assert np.all(oracle == 2.0)
    for backend in (X.Parallel(4), X.Graph(4)):
        g, a = build(True, True)
        g.run(backend)
        assert np.array_equal(g.copy_to_host(a), oracle)
        g, a = build(False, True)
        g.run(backend)
        assert np.all(g.copy_to_host(a) == 1.0)  # transform ran first on the other stream


@pytest.mark.gpu
@gpu
@pytest.mark.parametrize("engine", ["philox", "mrg"])
def test_generate_transform_chain_matches_oracle_on_every_backend(engine):
    from oracle import oracle as O

    kind = P.EngineKind.PHILOX4X32X10 if engine == "philox" else P.EngineKind.MRG32K3A
    n = 100003

    def run(backend, gauss=False):
        g = X.TaskGraph()
        buf = g.create_buffer(n, "f32")
        st = P.seed_engine(kind, 42)
        gen = (X.gaussian_generate_kernel(st, buf.id, 0.0, 1.0, "fp32") if gauss
               else X.uniform_generate_kernel(st, buf.id, "fp32"))
        g.submit_with_accessors(gen, [(buf, RW)])
        g.submit_with_accessors(X.affine_kernel(buf.id, -1.0, 1.0), [(buf, RW)])
        g.run(backend)
        return g.copy_to_host(buf)

    if engine == "philox":
        words = O.philox_words(O.seed_philox(42), 0, n)
    else:
        s1, s2 = O.seed_mrg(42)
        words = O.mrg_fill(*s1, *s2, n)[0]
    want = O.range_transform(O.words_to_unit(words, "fp32"), -1.0, 1.0)
    serial = run(X.Serial())
    assert np.array_equal(serial, want)
    gs = run(X.Serial(), gauss=True)
    for backend in BACKENDS[1:]:
        assert np.array_equal(run(backend), serial), backend
        assert np.array_equal(run(backend, gauss=True), gs), backend  # odd chunk starts re-pair


def _random_graph(rng, tasks=None):
    """Random accessor-declared DAG of elementwise kernels (test_execution.py:156-187)."""
    g = X.TaskGraph()
    length = int(rng.integers(1, 600))
    buffers = [g.create_buffer(length) for _ in range(int(rng.integers(2, 5)))]
    for _ in range(tasks if tasks is not None else int(rng.integers(1, 21))):
        k = int(rng.integers(1, min(3, len(buffers)) + 1))
        chosen = rng.choice(len(buffers), size=k, replace=False)
        modes = [X.AccessMode(rng.choice(["read", "write", "read_write"])) for _ in chosen]
        if not any(m in (W, RW) for m in modes):
            modes[0] = RW
        coef, bias = float(rng.uniform(0.5, 1.5)), float(rng.uniform(-1.0, 1.0))
        handles = [buffers[int(i)] for i in chosen]

        def kernel(views, start, stop, handles=handles, modes=modes, coef=coef, bias=bias):
            reads = [views[h.id][start:stop].clone() for h, m in zip(handles, modes) if m in (R, RW)]
            for h, m in zip(handles, modes):
                if m in (W, RW):
                    seg = views[h.id][start:stop]
                    seg *= coef
                    seg += bias
                    for r in reads:
                        seg += r

        g.submit_with_accessors(kernel, list(zip(handles, modes)))
    return g, buffers


@pytest.mark.gpu
@gpu
def test_random_graphs_all_backends_equal_serial_and_start_topologically():
    rng = np.random.default_rng(11)
    for _ in range(8):
        seed = int(rng.integers(0, 2 ** 31))
        results = []
        for backend in BACKENDS:
            g, buffers = _random_graph(np.random.default_rng(seed))
            report = g.run(backend)
            times = {t.task_id: t for t in report.tasks}
            for u, v in g.edges:
                assert times[v].start_ns >= times[u].end_ns - 1000, backend  # event clock: ~0.5 us
            results.append([g.copy_to_host(b) for b in buffers])
        for other in results[1:]:
            for a, b in zip(results[0], other):
                assert np.array_equal(a, b)


@pytest.mark.gpu
@gpu
def test_chunk_coverage_unsplittable_and_panic():
    for backend in (X.Serial(), X.Parallel(3, chunk=7), X.Graph(8)):
        g = X.TaskGraph()
        a = g.create_buffer(1001)

        def probe(views, start, stop):
            views[a.id][start:stop] += 1.0

        g.submit_with_accessors(probe, [(a, RW)])
        g.run(backend)
        assert np.all(g.copy_to_host(a) == 1.0)
    g = X.TaskGraph()
    a = g.create_buffer(10000)
    calls = []

    def kernel(views, start, stop):
        calls.append((start, stop))
        views[a.id][start:stop] = 1.0

    g.submit_with_accessors(kernel, [(a, RW)], splittable=False)
    g.run(X.Parallel(8))
    assert calls == [(0, 10000)]

    def boom(views, start, stop):
        raise RuntimeError("exploded")

    for backend in (X.Serial(), X.Parallel(2)):
        g = X.TaskGraph()
        a = g.create_buffer(16)
        ev = g.submit_with_accessors(boom, [(a, RW)])
        with pytest.raises(X.KernelPanic, match=f"task {ev.task_id}"):
            g.run(backend)
