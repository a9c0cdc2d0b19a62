"""prng_calo_deposit (csrc/calo.cu calo_deposit_kernel) against numpy's own
np.unique + np.bincount -- the reference's per-event deposition
(calosim.py:340-347) -- on adversarial events: empty events, one hit, warp
boundaries, every hit in one cell, a few hot cells, more unique cells than
one walk holds, cell ranges wider than one bitmap window (and ids near
2^32), and amounts whose sums depend on the addition order.  Bit-exact.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _numpy_deposits(cells, amts, offs):
    out_c, out_e, counts = [], [], []
    for e in range(len(offs) - 1):
        c = cells[offs[e]:offs[e + 1]]
        a = amts[offs[e]:offs[e + 1]]
        if len(c) == 0:
            counts.append(0)
            continue
        u, inv = np.unique(c, return_inverse=True)
        out_c.append(u)
        out_e.append(np.bincount(inv, weights=a))
        counts.append(len(u))
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt)  # noqa: E731
    return cat(out_c, np.uint32), cat(out_e, np.float64), np.asarray(counts, dtype=np.int64)


def _events(rng):
    """(cells, amounts) per event covering the kernel's edge cases."""
    ev = []
    mag = lambda n: rng.choice([1.0, 1e-3, 1e8, 3e15], size=n) * rng.random(n)  # noqa: E731
    ev.append((np.zeros(0, np.uint32), np.zeros(0)))                       # empty
    ev.append((np.array([7], np.uint32), np.array([0.5])))                 # one hit
    for n in (31, 32, 33, 64, 65):                                          # warp boundaries
        ev.append((rng.integers(0, 50, n).astype(np.uint32), mag(n)))
    ev.append((np.full(5000, 123456, np.uint32), mag(5000)))               # one cell
    ev.append((rng.choice(np.array([5, 9, 190000 - 1], np.uint32), 3000), mag(3000)))  # hot cells
    ev.append((rng.integers(0, 190000, 20000).astype(np.uint32), mag(20000)))  # > 4096 unique cells
    ev.append((np.arange(9000, dtype=np.uint32)[::-1].copy(), mag(9000)))  # all unique, descending
    ev.append((np.array([0, 1 << 18, (1 << 18) - 1, 1 << 20, 3, 1 << 18], np.uint32), mag(6)))  # > 1 window
    ev.append((np.array([0xFFFFFFFF, 0, 0xFFFFFFF0, 0xFFFFFFFF, 77], np.uint32), mag(5)))   # ids near 2^32
    ev.append((rng.integers(0, 1 << 20, 4000).astype(np.uint32), mag(4000)))  # several windows
    ev.append((np.zeros(0, np.uint32), np.zeros(0)))                       # empty again
    for _ in range(40):                                                     # ordinary events
        n = int(rng.integers(0, 600))
        ev.append((rng.integers(1000, 9000, n).astype(np.uint32), mag(n)))
    return ev


def _run(lib, torch, cells, amts, offs, cell_bits):
    nev = len(offs) - 1
    total = int(offs[-1])
    d_cells = torch.from_numpy(cells.view(np.int32)).cuda()
    d_amts = torch.from_numpy(amts).cuda()
    d_offs = torch.from_numpy(offs.astype(np.int64)).cuda()
    nbytes = lib.prng_calo_deposit_scratch_bytes(total, nev)
    scratch = torch.full((max(nbytes, 1),), 0xAB, dtype=torch.uint8, device="cuda")  # dirty: the call zeroes it
    dep_c = torch.zeros(max(total, 1), dtype=torch.int32, device="cuda")
    dep_e = torch.zeros(max(total, 1), dtype=torch.float64, device="cuda")
    dep_o = torch.zeros(nev + 1, dtype=torch.int64, device="cuda")
    from paper_2109_01329_b200 import _lib
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.prng_calo_deposit(d_cells.data_ptr(), d_amts.data_ptr(), total, d_offs.data_ptr(), nev, cell_bits,
                                     scratch.data_ptr(), nbytes, dep_c.data_ptr(), dep_e.data_ptr(),
                                     dep_o.data_ptr(), s))
    torch.cuda.synchronize()
    o = dep_o.cpu().numpy()
    n = int(o[-1])
    return dep_c.cpu().numpy().view(np.uint32)[:n], dep_e.cpu().numpy()[:n], o


@pytest.mark.parametrize("seed", [1, 2])
def test_deposit_matches_numpy_unique_bincount(seed):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2109_01329_b200 import _lib
    rng = np.random.default_rng(seed)
    ev = _events(rng)
    order = rng.permutation(len(ev)) if seed == 2 else np.arange(len(ev))
    ev = [ev[i] for i in order]
    cells = np.concatenate([c for c, _ in ev]).astype(np.uint32)
    amts = np.concatenate([a for _, a in ev]).astype(np.float64)
    offs = np.zeros(len(ev) + 1, dtype=np.int64)
    np.cumsum([len(c) for c, _ in ev], out=offs[1:])
    want_c, want_e, counts = _numpy_deposits(cells, amts, offs)
    for cell_bits in (32, 0):
        got_c, got_e, got_o = _run(_lib.lib, torch, cells, amts, offs, cell_bits)
        assert np.array_equal(np.diff(got_o), counts)
        assert np.array_equal(got_c, want_c)
        assert np.array_equal(got_e.view(np.uint64), want_e.view(np.uint64))


def test_deposit_small_cell_bits_and_many_events():
    """Narrow window (cell_bits 10) and more events than resident CTAs: the
    look-back chains across thousands of tickets."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2109_01329_b200 import _lib
    rng = np.random.default_rng(5)
    nev = 5000
    counts_h = rng.integers(0, 80, nev)
    offs = np.zeros(nev + 1, dtype=np.int64)
    np.cumsum(counts_h, out=offs[1:])
    cells = rng.integers(0, 1 << 10, int(offs[-1])).astype(np.uint32)
    amts = rng.random(int(offs[-1])) * rng.choice([1.0, 1e12], int(offs[-1]))
    want_c, want_e, counts = _numpy_deposits(cells, amts, offs)
    got_c, got_e, got_o = _run(_lib.lib, torch, cells, amts, offs, 10)
    assert np.array_equal(np.diff(got_o), counts)
    assert np.array_equal(got_c, want_c)
    assert np.array_equal(got_e.view(np.uint64), want_e.view(np.uint64))


def test_deposit_narrow_ids_and_bucket_storage():
    """Ids below 2^cell_bits with cell_bits <= 18 (one window from 0, no
    min/max pass): empty, single-hit, exactly-8192-hit (the largest event
    with shared-memory buckets) next to 8193-hit (32-bit buckets in scratch),
    hot-cell (> 32 hits per bucket: the CTA-wide bitonic order) and
    all-unique events; the same events again with cell_bits = 0."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2109_01329_b200 import _lib
    rng = np.random.default_rng(11)
    mag = lambda n: rng.choice([1.0, 1e-3, 1e8, 3e15], size=n) * rng.random(n)  # noqa: E731
    ev = [(np.zeros(0, np.uint32), np.zeros(0)), (np.array([5], np.uint32), np.array([2.5]))]
    ev.append((rng.integers(0, 1 << 18, 8192).astype(np.uint32), mag(8192)))
    ev.append((rng.integers(0, 1 << 18, 8193).astype(np.uint32), mag(8193)))
    ev.append((rng.choice(np.array([7, 70000, (1 << 18) - 1], np.uint32), 4000), mag(4000)))
    ev.append((np.full(3000, 12345, np.uint32), mag(3000)))
    ev.append((rng.permutation(6000).astype(np.uint32) * 41, mag(6000)))
    for _ in range(300):
        n = int(rng.integers(0, 300))
        ev.append((rng.integers(0, 1 << 18, n).astype(np.uint32), mag(n)))
    cells = np.concatenate([c for c, _ in ev]).astype(np.uint32)
    amts = np.concatenate([a for _, a in ev]).astype(np.float64)
    offs = np.zeros(len(ev) + 1, dtype=np.int64)
    np.cumsum([len(c) for c, _ in ev], out=offs[1:])
    want_c, want_e, counts = _numpy_deposits(cells, amts, offs)
    for cell_bits in (18, 0):
        got_c, got_e, got_o = _run(_lib.lib, torch, cells, amts, offs, cell_bits)
        assert np.array_equal(np.diff(got_o), counts)
        assert np.array_equal(got_c, want_c)
        assert np.array_equal(got_e.view(np.uint64), want_e.view(np.uint64))


def test_deposit_understated_cell_bits_is_detected():
    """cell_bits is a performance hint: ids at or above 2^cell_bits (an
    understated bound) are detected per event and the event is redone over
    min/max windows, so the deposits are still numpy's."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2109_01329_b200 import _lib
    rng = np.random.default_rng(17)
    ev = [(rng.integers(0, 1 << 10, 500).astype(np.uint32), rng.random(500)),        # inside 2^10
          (rng.integers(0, 1 << 18, 3000).astype(np.uint32), rng.random(3000)),      # mostly outside
          (np.array([1023, 1024, 5, 1 << 31], np.uint32), rng.random(4)),            # straddles, and far
          (np.zeros(0, np.uint32), np.zeros(0))]
    cells = np.concatenate([c for c, _ in ev]).astype(np.uint32)
    amts = np.concatenate([a for _, a in ev]).astype(np.float64)
    offs = np.zeros(len(ev) + 1, dtype=np.int64)
    np.cumsum([len(c) for c, _ in ev], out=offs[1:])
    want_c, want_e, counts = _numpy_deposits(cells, amts, offs)
    got_c, got_e, got_o = _run(_lib.lib, torch, cells, amts, offs, 10)
    assert np.array_equal(np.diff(got_o), counts)
    assert np.array_equal(got_c, want_c)
    assert np.array_equal(got_e.view(np.uint64), want_e.view(np.uint64))
