"""FastCaloSim RNG consumption (calosim.py:269-358): planning and batches.

CPU part: the host bookkeeping (hits, allocations, position chain) driven by
oracle control draws must reproduce the reference's simulate_event numbers
(golden.json "calosim").  GPU part: plan_events, the segment kernel and the
CUDA-graph replay reproduce the same batches as per-batch generation and the
oracle stream.
"""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2109_01329_b200 import calosim as C


def _oracle_draws(key):
    def batched(positions, counts):
        parts = [O.words_to_unit(O.philox_words(key, p, c), "fp32").astype(np.float64)
                 for p, c in zip(positions, counts)]
        return np.concatenate(parts) if parts else np.zeros(0)

    def one(position, count):
        return O.words_to_unit(O.philox_words(key, position, count), "fp32").astype(np.float64)

    return batched, one


@pytest.mark.parametrize("label", ["electron", "ttbar_small_batch"])
def test_plan_matches_reference_simulate_event(golden, label):
    ref = golden["calosim"][label]
    ranges = [[tuple(r) for r in e["hit_ranges"]] for e in ref["events"]]
    hits, allocs = C.plan_from_controls(0, ranges, ref["min_batch"], *_oracle_draws(O.seed_philox(777)))
    assert hits == [e["hits"] for e in ref["events"]]
    assert allocs == [e["allocated"] for e in ref["events"]]
    assert sum(allocs) == ref["final_position"]


def test_batches_start_where_reference_batches_start(golden):
    ref = golden["calosim"]["electron"]
    key = O.seed_philox(777)
    pos = 0
    for e in ref["events"]:
        assert O.words_to_unit(O.philox_words(key, pos, 4), "fp32").tolist() == e["first4"]
        pos += e["allocated"]


@pytest.mark.parametrize("label", ["electron", "ttbar_small_batch"])
def test_cpu_deposition_oracle_matches_reference(golden, golden_arrays, label):
    """oracle/calo_cpu.py (the C5 CPU baseline) reproduces the reference's
    simulate_event deposits from oracle-generated batches."""
    from oracle import calo_cpu

    ref = golden["calosim"][label]
    nreg = len([k for k in golden_arrays if k.startswith("calo_geom__")])
    geom = [golden_arrays[f"calo_geom__{r:02d}"] for r in range(nreg)]
    params = {k: (np.asarray(v["bin_edges"]), np.asarray(v["weights"])) for k, v in ref["params"].items()}
    key = O.seed_philox(777)
    ranges = [[tuple(r) for r in e["hit_ranges"]] for e in ref["events"]]
    pp = []
    C.plan_from_controls(0, ranges, ref["min_batch"], *_oracle_draws(key), per_particle=pp)
    pos = 0
    for e, ev in enumerate(ref["events"][:6]):
        batch = O.words_to_unit(O.philox_words(key, pos, ev["allocated"]), "fp32")
        dep, psums = calo_cpu.deposit_event(batch, ev["particles"], pp[e], geom, params, nreg,
                                            ref["sampling_fraction"])
        assert psums == ev["particle_sums"]
        cells = golden_arrays[f"calo__{label}__{e:03d}__cells"]
        assert sorted(dep) == cells.tolist()
        assert [dep[c] for c in cells.tolist()] == golden_arrays[f"calo__{label}__{e:03d}__sums"].tolist()
        pos += ev["allocated"]


@pytest.mark.gpu
@pytest.mark.parametrize("label", ["electron", "ttbar_small_batch"])
def test_gpu_deposition_bit_identical_to_reference(golden, golden_arrays, label):
    """simulate_events (control draws, one segment launch, hit kernel,
    pairwise normalisation, deposit kernel) == the reference's
    simulate_event deposits, particle sums and accounting, exactly."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2109_01329_b200 as P

    ref = golden["calosim"][label]
    nreg = len([k for k in golden_arrays if k.startswith("calo_geom__")])
    geom = [golden_arrays[f"calo_geom__{r:02d}"] for r in range(nreg)]
    params = {k: C.Parameterization(k, v["hit_lo"], v["hit_hi"], v["bin_edges"], v["weights"])
              for k, v in ref["params"].items()}
    det = C.Detector(geom, params)
    events = [[C.Particle(k, e, tuple(d)) for k, e, d in ev["particles"]] for ev in ref["events"]]
    st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
    final, results = C.simulate_events(events, det, st, ref["min_batch"], ref["sampling_fraction"])
    assert P.stream_position(final) == ref["final_position"]
    for e, (res, want) in enumerate(zip(results, ref["events"])):
        assert res.hits == want["hits"] and res.randoms_allocated == want["allocated"]
        assert res.particle_sums == want["particle_sums"], e
        cells = golden_arrays[f"calo__{label}__{e:03d}__cells"]
        sums = golden_arrays[f"calo__{label}__{e:03d}__sums"]
        assert sorted(res.deposits) == cells.tolist(), e
        assert [res.deposits[c] for c in cells.tolist()] == sums.tolist(), e


@pytest.mark.gpu
def test_gpu_plan_segments_and_graph(golden):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2109_01329_b200 as P

    for label in ("electron", "ttbar_small_batch"):
        ref = golden["calosim"][label]
        ranges = [[tuple(r) for r in e["hit_ranges"]] for e in ref["events"]]
        st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
        hits, allocs, table, final = C.plan_events(st, ranges, ref["min_batch"])
        assert hits == [e["hits"] for e in ref["events"]]
        assert allocs == [e["allocated"] for e in ref["events"]]
        assert P.stream_position(final) == ref["final_position"]
        total = sum(allocs)
        seg = torch.empty(total, dtype=torch.float32, device="cuda")
        C.generate_segments(st, table, seg)
        eager = torch.empty_like(seg)
        C.per_batch(st, allocs, eager)
        g = C.BatchGraph(st, allocs, torch.zeros_like(seg))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(seg, eager) and torch.equal(g.out, eager)
        want = O.words_to_unit(O.philox_words(O.seed_philox(777), 0, total), "fp32")
        assert np.array_equal(seg.cpu().numpy(), want)
        off = 0
        for e in ref["events"]:
            assert seg[off:off + 4].cpu().tolist() == e["first4"]
            off += e["allocated"]


@pytest.mark.gpu
@pytest.mark.parametrize("label", ["electron", "ttbar_small_batch"])
def test_gpu_chunking_does_not_change_results(golden, golden_arrays, label):
    """simulate_events' chunked pipeline (array planning per chunk, the
    event-by-event fallback where a chunk's positions depend on its hits)
    gives the same packed deposits, sums and final state for any chunk size."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2109_01329_b200 as P

    ref = golden["calosim"][label]
    nreg = len([k for k in golden_arrays if k.startswith("calo_geom__")])
    geom = [golden_arrays[f"calo_geom__{r:02d}"] for r in range(nreg)]
    params = {k: C.Parameterization(k, v["hit_lo"], v["hit_hi"], v["bin_edges"], v["weights"])
              for k, v in ref["params"].items()}
    det = C.Detector(geom, params)
    events = [[C.Particle(k, e, tuple(d)) for k, e, d in ev["particles"]] for ev in ref["events"]]
    events = events * 3 + [[]] + events[:2]  # more events than one chunk, and an empty event
    st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
    runs = [C.simulate_events(events, det, st, ref["min_batch"], ref["sampling_fraction"], dicts=False,
                              chunk_events=k) for k in (1, 3, 7, 2048)]
    f0, r0 = runs[0]
    for f, r in runs[1:]:
        assert P.stream_position(f) == P.stream_position(f0)
        for key in ("cells", "energy", "counts", "offsets", "particle_sums"):
            assert np.array_equal(r[key], r0[key]), key
        assert r["hits"] == r0["hits"] and r["allocated"] == r0["allocated"]
    with pytest.raises(P.InvalidParameter):
        C.simulate_events([[C.Particle("muon", 1.0, (0.0, 0.0, 1.0))]], det, st)


@pytest.mark.gpu
def test_gpu_pairwise_normalisation_all_tree_shapes():
    """Particles from < 8 hits (one short leaf) through one full leaf, a few
    leaves, and trees too large for the listed path (> 256 leaves: lane 0
    sums them on the fly) -- GPU simulate_events against the CPU oracle's
    simulate_event restatement on the same oracle-generated batches: particle
    sums (numpy pairwise, bit for bit) and deposits."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2109_01329_b200 as P
    from oracle import calo_cpu

    nreg = 4
    geom = [np.arange(r, 4000, nreg, dtype=np.int64) for r in range(nreg)]
    edges = np.linspace(0.001, 0.101, 9)
    weights = np.asarray([0.05, 0.10, 0.20, 0.25, 0.20, 0.10, 0.07, 0.03])
    ranges = {"tiny": (1, 7), "leaf": (8, 128), "few": (129, 700), "huge": (33000, 40000)}
    det = C.Detector(geom, {k: C.Parameterization(k, lo, hi, edges, weights) for k, (lo, hi) in ranges.items()})
    rng = np.random.default_rng(3)
    kinds = list(ranges)
    events = []
    for e in range(12):
        parts = [C.Particle(kinds[(e + j) % 4], float(rng.uniform(1.0, 50.0)),
                            tuple(rng.normal(size=3) / np.sqrt(3))) for j in range(1 + e % 3)]
        events.append(parts)
    min_batch, sf = 1000, 0.8
    st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
    final, results = C.simulate_events(events, det, st, min_batch, sf)
    key = O.seed_philox(777)
    pp = []
    hits, allocs = C.plan_from_controls(0, [[ranges[p.kind] for p in ev] for ev in events], min_batch,
                                        *_oracle_draws(key), per_particle=pp)
    params = {k: (edges, weights) for k in ranges}
    pos = 0
    for e, ev in enumerate(events):
        batch = O.words_to_unit(O.philox_words(key, pos, allocs[e]), "fp32")
        dep, psums = calo_cpu.deposit_event(batch, [(p.kind, p.energy, p.direction) for p in ev], pp[e], geom,
                                            params, nreg, sf)
        assert results[e].hits == hits[e] and results[e].particle_sums == psums, e
        assert results[e].deposits == dep, e
        pos += allocs[e]
    assert P.stream_position(final) == pos
