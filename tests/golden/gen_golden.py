#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/gen_golden.py [--reference /root/reference]

It imports `portarng` from /root/reference/pkg/src.  When oracle/_ref holds
the reference's compiled Cython core (oracle/build_ref.sh) it is installed
as `portarng._kernels._core`, so the fixtures come from the same native code
the reference ships (otherwise the reference's numpy fallback is used; the
integer streams are bit-identical either way, _kernels/_fallback.py:1-7).

Outputs (small, committed):
  golden.json  -- KATs, first words, sha256[:16] hashes of large streams,
                  MRG jump-ahead states, lognormal definition vectors
  cases.npz    -- arrays for every parity case in CASES below
The GPU box never runs this script (no /root/reference there).
"""

from __future__ import annotations

import argparse
import hashlib
import importlib.util
import json
import math
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent


def sha16(arr):
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()[:16]


def load_reference(root: Path):
    sys.path.insert(0, str(root / "pkg" / "src"))
    sys.path.insert(0, str(root / "pkg" / "tests"))
    core_impl = "fallback"
    ref_dir = REPO / "oracle" / "_ref"
    if ref_dir.is_dir() and os.environ.get("PORTARNG_KERNELS") != "fallback":
        for f in ref_dir.iterdir():
            if f.name.startswith("_core") and f.suffix == ".so":
                spec = importlib.util.spec_from_file_location("portarng._kernels._core", f)
                mod = importlib.util.module_from_spec(spec)
                spec.loader.exec_module(mod)
                sys.modules["portarng._kernels._core"] = mod
                core_impl = "core"
    import portarng  # noqa: F401
    from portarng import _kernels

    assert _kernels.IMPL == core_impl, (_kernels.IMPL, core_impl)
    return core_impl


# Parity cases: (name, engine, seed, skip, dist, precision, p0, p1, n)
#  engine 'philox' | 'mrg'; skip = words skipped before generating (Philox
#  only in the reference); dist 'bits' | 'uniform' | 'gaussian' | 'lognormal'.
CASES = []
for n in (0, 1, 3, 4, 5, 64, 1001, 4097):
    CASES.append((f"philox_bits_n{n}", "philox", 2024, 0, "bits", "fp32", 0, 0, n))
    CASES.append((f"mrg_bits_n{n}", "mrg", 2024, 0, "bits", "fp32", 0, 0, n))
for skip in (1, 2, 3, 5, 6, 7, 1000003):
    CASES.append((f"philox_bits_skip{skip}", "philox", 0xCAFEF00D12345678, skip, "bits", "fp32", 0, 0, 1031))
    CASES.append((f"philox_u32_skip{skip}", "philox", 777, skip, "uniform", "fp32", 0.0, 1.0, 1031))
    CASES.append((f"philox_g32_skip{skip}", "philox", 777, skip, "gaussian", "fp32", 0.0, 1.0, 1031))
    CASES.append((f"philox_g64_skip{skip}", "philox", 777, skip, "gaussian", "fp64", 2.0, 0.5, 1030))
for lo, hi in ((0.0, 1.0), (-1.0, 1.0), (-123.456, 987.654), (1e-3, 2e-3), (-5e5, 3.25)):
    for prec in ("fp32", "fp64"):
        tag = f"{lo:g}_{hi:g}_{prec}"
        CASES.append((f"philox_uniform_{tag}", "philox", 777, 0, "uniform", prec, lo, hi, 4099))
        CASES.append((f"mrg_uniform_{tag}", "mrg", 777, 0, "uniform", prec, lo, hi, 4099))
for mean, sd in ((0.0, 1.0), (2.0, 0.5), (-7.5, 3.0), (1e4, 1e-2)):
    for prec in ("fp32", "fp64"):
        for n in (4096, 4095):
            tag = f"{mean:g}_{sd:g}_{prec}_n{n}"
            CASES.append((f"philox_gauss_{tag}", "philox", 1618033, 0, "gaussian", prec, mean, sd, n))
            CASES.append((f"mrg_gauss_{tag}", "mrg", 1618033, 0, "gaussian", prec, mean, sd, n))
for m, s in ((0.0, 1.0), (1.5, 0.25), (-2.0, 0.75)):
    for prec in ("fp32", "fp64"):
        tag = f"{m:g}_{s:g}_{prec}"
        CASES.append((f"philox_lognorm_{tag}", "philox", 4242, 0, "lognormal", prec, m, s, 2049))
        CASES.append((f"mrg_lognorm_{tag}", "mrg", 4242, 0, "lognormal", prec, m, s, 2049))


def run_case(case):
    from portarng import distributions as D
    from portarng.engine import EngineKind, generate_words, seed_engine, skip_ahead

    name, engine, seed, skip, dist, prec, p0, p1, n = case
    kind = EngineKind.PHILOX4X32X10 if engine == "philox" else EngineKind.MRG32K3A
    state = seed_engine(kind, seed)
    if skip:
        state = skip_ahead(state, skip)
    if dist == "bits":
        return generate_words(state, n)[1]
    if dist == "uniform":
        _, block = D.fill_uniform_unit(state, n, prec)
        return D.range_transform(block, p0, p1).values
    if dist == "gaussian":
        return D.fill_gaussian(state, n, p0, p1, prec)[1].values
    # lognormal extension: exp (libm, via math.exp) of the reference's fp64
    # Box-Muller variate m + s*z, then cast.
    _, words = generate_words(state, 2 * ((n + 1) // 2))
    z = D.gaussian_from_words(words, p0, p1, n, "fp64")
    x = np.array([math.exp(v) for v in z], dtype=np.float64)
    return x.astype(np.float32 if prec == "fp32" else np.float64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reference", default="/root/reference")
    args = ap.parse_args()
    impl = load_reference(Path(args.reference))

    from oracles import PHILOX_KAT
    from portarng import distributions as D
    from portarng.engine import EngineKind, generate_words, next_word, seed_engine, skip_ahead
    from portarng.execution import Parallel, Serial
    from portarng.rngburn import burn_once

    P, M = EngineKind.PHILOX4X32X10, EngineKind.MRG32K3A
    g = {"generated_with": {"reference": args.reference, "kernel_impl": impl,
                            "numpy": np.__version__}}
    g["philox_kat"] = [[list(k), list(c), list(e)] for k, c, e in PHILOX_KAT]

    s777 = seed_engine(P, 777)
    _, w = generate_words(s777, 1 << 24)
    g["philox777_words8"] = [int(x) for x in w[:8]]
    g["philox777_u32_2p24_sha16"] = sha16(w)
    _, blk = D.fill_uniform_unit(s777, 1 << 24, "fp32")
    g["philox777_uniform_f32_2p24_sha16"] = sha16(D.range_transform(blk, 0.0, 1.0).values)
    g["philox777_uniform_f32_first4"] = [float(x) for x in blk.values[:4]]
    _, blk = D.fill_uniform_unit(s777, 1 << 20, "fp64")
    g["philox777_uniform_f64_m1p1_2p20_sha16"] = sha16(D.range_transform(blk, -1.0, 1.0).values)
    gz = D.fill_gaussian(s777, 1 << 20, 0.0, 1.0, "fp32")[1].values
    g["philox777_gauss_f32_2p20_sha16"] = sha16(gz)
    # Position-independent window checks at a far offset (calosim substreams sit at 2**96).
    far = skip_ahead(s777, (1 << 98) + 3)
    g["philox777_far_2p98p3_words16"] = [int(x) for x in generate_words(far, 16)[1]]

    m777 = seed_engine(M, 777)
    _, mw = generate_words(m777, 1 << 20)
    g["mrg777_words4"] = [int(x) for x in mw[:4]]
    g["mrg777_word_2p20m1"] = int(mw[-1])
    g["mrg777_u32_2p20_sha16"] = sha16(mw)
    _, blk = D.fill_uniform_unit(m777, 1 << 20, "fp64")
    mu = D.range_transform(blk, -1.0, 1.0).values
    g["mrg777_uniform_f64_m1p1_2p20_sha16"] = sha16(mu)
    g["mrg777_uniform_f64_first2"] = [float(x) for x in mu[:2]]
    # MRG hand values (test_engine.py:78-84)
    st, z = next_word(seed_engine(M, 0))
    g["mrg_seed0_step1"] = {"s1": list(st.s1), "s2": list(st.s2), "z": int(z)}
    # Jump-ahead pins: windows after k sequential steps of the reference core.
    jumps = {}
    for seed in (777, 12345, 2**63 + 5):
        base = seed_engine(M, seed)
        for k in (1, 2, 3, 5, 1000, 123457, 1 << 20):
            s, _ = generate_words(base, k)
            jumps[f"{seed}:{k}"] = {"s1": list(s.s1), "s2": list(s.s2)}
    g["mrg_jumps"] = jumps

    # burn_once mode invariance outputs (test_rngburn.py:52-73) at small batches.
    burns = {}
    arrays = {}
    for label, eng, spec, batch, seed in (
        ("philox_uniform_m1p1_1000", P, D.Uniform(-1.0, 1.0), 1000, 99),
        ("mrg_uniform_m1p1_500", M, D.Uniform(-1.0, 1.0), 500, 99),
        ("philox_gauss_2_0.5_1001", P, D.Gaussian(2.0, 0.5), 1001, 7),
        ("philox_uniform_f64_m1p1_777", P, D.Uniform(-1.0, 1.0, "fp64"), 777, 13),
    ):
        out = burn_once(eng, spec, "buffer", Serial(), batch, seed)[1]
        par = burn_once(eng, spec, "usm", Parallel(4), batch, seed)[1]
        assert np.array_equal(out, par)
        arrays[f"burn__{label}"] = out
        burns[label] = sha16(out)
    g["burn_once_sha16"] = burns

    # FastCaloSim RNG consumption (calosim.simulate_event, calosim.py:269-358):
    # per-event hits, allocations and the first uniforms of each device batch.
    from portarng import calosim as C

    geo = C.synth_geometry(20000, C.DEFAULT_REGIONS)
    for r, ids in enumerate(geo.region_cell_ids):
        arrays[f"calo_geom__{r:02d}"] = np.asarray(ids, dtype=np.int64)
    calo = {}
    for label, scen, nev, min_batch, sf in (
            ("electron", C.ScenarioKind.SINGLE_ELECTRON, 40, C.DEFAULT_MIN_BATCH, 1.0),
            ("ttbar_small_batch", C.ScenarioKind.TTBAR, 3, 1000, 0.25)):
        params = C.synth_params(scen)
        evs = C._synth_events(scen, nev, 777, params)
        st = seed_engine(P, 777)
        rows = []
        for e, ev in enumerate(evs):
            st2, res = C.simulate_event(ev, geo, params, st, min_batch=min_batch, sampling_fraction=sf)
            first = D.fill_uniform_unit(st, 4, "fp32")[1].values
            rows.append({"hit_ranges": [[params[p.kind].hit_lo, params[p.kind].hit_hi] for p in ev.particles],
                         "particles": [[p.kind, p.energy, list(p.direction)] for p in ev.particles],
                         "hits": res.hits, "allocated": res.randoms_allocated,
                         "particle_sums": [float(x) for x in res.particle_sums],
                         "first4": [float(x) for x in first]})
            cells = np.asarray(sorted(res.deposits), dtype=np.int64)
            arrays[f"calo__{label}__{e:03d}__cells"] = cells
            arrays[f"calo__{label}__{e:03d}__sums"] = np.asarray([res.deposits[c] for c in cells.tolist()])
            st = st2
        calo[label] = {"min_batch": min_batch, "sampling_fraction": sf, "events": rows,
                       "final_position": int(__import__("portarng").engine.stream_position(st)),
                       "params": {k: {"hit_lo": p.hit_lo, "hit_hi": p.hit_hi, "bin_edges": p.bin_edges.tolist(),
                                      "weights": p.weights.tolist()} for k, p in params.items()}}
    g["calosim"] = calo

    # Burner result file format (rngburn.write_records_csv, rngburn.py:183-192).
    import tempfile

    from portarng.metrics import RunRecord as RefRecord
    from portarng.rngburn import write_records_csv

    recs = [RefRecord("b200", "buffer", "cuda:148sm", "philox", "uniform:-1:1", 1000, [1500, 1400, 1450]),
            RefRecord("b200", "usm", "cuda:148sm", "mrg32k3a", "gaussian:2:0.5", 7, [99])]
    with tempfile.NamedTemporaryFile("r", suffix=".csv") as tmp:
        write_records_csv(recs, tmp.name)
        g["burner_csv"] = open(tmp.name).read()

    for case in CASES:
        arrays[f"case__{case[0]}"] = run_case(case)
    g["cases"] = [list(c) for c in CASES]

    np.savez_compressed(HERE / "cases.npz", **arrays)
    (HERE / "golden.json").write_text(json.dumps(g, indent=1, sort_keys=True) + "\n")
    print(f"wrote {len(arrays)} arrays, impl={impl}")


if __name__ == "__main__":
    main()
