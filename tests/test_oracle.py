"""Pin the CPU oracle (oracle/) to the reference's golden vectors and core.

CPU-only.  These are the checks that make the oracle trustworthy before it is
used as the parity checker for the CUDA path (tests/test_gpu_parity.py).
"""

import numpy as np
import pytest

from oracle import oracle as O
from refcases import oracle_case


def test_philox_known_answers(golden):
    # tests/oracles.py:56-68 (Random123 zero / all-ones / pi-digits)
    for key, ctr, expected in golden["philox_kat"]:
        assert O.philox_block(tuple(key), tuple(ctr)) == tuple(expected)


def test_philox777_stream_hashes(golden):
    key = O.seed_philox(777)
    w = O.philox_words(key, 0, 1 << 24)
    assert [int(x) for x in w[:8]] == golden["philox777_words8"]
    assert O.sha16(w) == golden["philox777_u32_2p24_sha16"]
    u = O.words_to_unit(w, "fp32")
    assert O.sha16(O.range_transform(u, 0.0, 1.0)) == golden["philox777_uniform_f32_2p24_sha16"]
    assert u[:4].tolist() == golden["philox777_uniform_f32_first4"]


def test_philox777_far_offset(golden):
    key = O.seed_philox(777)
    assert O.philox_words(key, (1 << 98) + 3, 16).tolist() == golden["philox777_far_2p98p3_words16"]


def test_philox_other_hashes(golden):
    key = O.seed_philox(777)
    u = O.generate("philox", (key, 0), "uniform", 1 << 20, "fp64", -1.0, 1.0)
    assert O.sha16(u) == golden["philox777_uniform_f64_m1p1_2p20_sha16"]
    z = O.generate("philox", (key, 0), "gaussian", 1 << 20, "fp32", 0.0, 1.0)
    assert O.sha16(z) == golden["philox777_gauss_f32_2p20_sha16"]


def test_mrg777_hashes(golden):
    s1, s2 = O.seed_mrg(777)
    w, _, _ = O.mrg_fill(*s1, *s2, 1 << 20)
    assert w[:4].tolist() == golden["mrg777_words4"]
    assert int(w[-1]) == golden["mrg777_word_2p20m1"]
    assert O.sha16(w) == golden["mrg777_u32_2p20_sha16"]
    u = O.generate("mrg", (s1, s2), "uniform", 1 << 20, "fp64", -1.0, 1.0)
    assert O.sha16(u) == golden["mrg777_uniform_f64_m1p1_2p20_sha16"]
    assert u[:2].tolist() == golden["mrg777_uniform_f64_first2"]


def test_mrg_seed0_hand_values(golden):
    # test_engine.py:78-84
    s1, s2 = O.seed_mrg(0)
    w, n1, n2 = O.mrg_fill(*s1, *s2, 1)
    ref = golden["mrg_seed0_step1"]
    assert list(n1) == ref["s1"] and list(n2) == ref["s2"] and int(w[0]) == ref["z"]


def test_mrg_jump_ahead_matches_sequential_reference(golden):
    # Extension a19 pinned on the reference's own sequential core.
    for key, want in golden["mrg_jumps"].items():
        seed, k = (int(x) for x in key.split(":"))
        s1, s2 = O.seed_mrg(seed)
        j1, j2 = O.mrg_skip(s1, s2, k)
        assert list(j1) == want["s1"] and list(j2) == want["s2"], key


def test_mrg_jump_composes():
    s1, s2 = O.seed_mrg(31337)
    a = O.mrg_skip(*O.mrg_skip(s1, s2, 12345), 67890)
    b = O.mrg_skip(s1, s2, 12345 + 67890)
    assert a == b
    # a jump of 2**127 + 2**64 + 3 composes the same way in the 128-bit form
    big = (1 << 127) + (1 << 64) + 3
    c = O.mrg_skip(*O.mrg_skip(s1, s2, big), 5)
    d = O.mrg_skip(s1, s2, big + 5)
    assert c == d


def test_all_golden_cases(golden, golden_arrays):
    for case in golden["cases"]:
        want = golden_arrays[f"case__{case[0]}"]
        got = oracle_case(case)
        assert got.dtype == want.dtype, case[0]
        assert np.array_equal(got, want), case[0]


def test_burn_once_outputs(golden_arrays):
    # rngburn.burn_once buffer/usm/Parallel outputs == whole-stream requests
    cases = {
        "philox_uniform_m1p1_1000": ("philox", (O.seed_philox(99), 0), "uniform", 1000, "fp32", -1.0, 1.0),
        "mrg_uniform_m1p1_500": ("mrg", O.seed_mrg(99), "uniform", 500, "fp32", -1.0, 1.0),
        "philox_gauss_2_0.5_1001": ("philox", (O.seed_philox(7), 0), "gaussian", 1001, "fp32", 2.0, 0.5),
        "philox_uniform_f64_m1p1_777": ("philox", (O.seed_philox(13), 0), "uniform", 777, "fp64", -1.0, 1.0),
    }
    for label, args in cases.items():
        got = O.generate(*args)
        want = golden_arrays[f"burn__{label}"]
        if args[2] == "gaussian":
            # burn_once applies the identity affine (rngburn.py:103-108) after generation
            got = O.range_transform(got, 0.0, 1.0)
        assert np.array_equal(got, want), label


def test_restatement_matches_reference_core():
    core = O.ref_core()
    if core is None:
        pytest.skip("oracle/_ref not built (oracle/build_ref.sh)")
    rng = np.random.default_rng(17)
    for _ in range(25):
        k0, k1 = (int(x) for x in rng.integers(0, 2**32, 2))
        b = [int(x) for x in rng.integers(0, 2**32, 4)]
        off = int(rng.integers(0, 4))
        n = int(rng.integers(1, 3000))
        assert np.array_equal(core.philox_fill(k0, k1, *b, off, n), O.philox_fill(k0, k1, *b, off, n))
    a, a1, a2 = core.mrg_fill(*(12345,) * 6, 5000)
    f, f1, f2 = O.mrg_fill(*(12345,) * 6, 5000)
    assert np.array_equal(a, f) and tuple(a1) == f1 and tuple(a2) == f2
    u1 = 1.0 - rng.integers(0, 2**24, 20000).astype(np.float64) / 2**24
    u2 = rng.integers(0, 2**24, 20000).astype(np.float64) / 2**24
    c0, c1 = core.box_muller(u1, u2)
    o0, o1 = O.box_muller(u1, u2)
    assert np.array_equal(c0, o0) and np.array_equal(c1, o1)


def test_cpu_baseline_cycles_match_oracle():
    """bench.py's cpu_baseline legs (reference core, chunked threads) produce
    the oracle's stream: uniform fp32, MRG fp64 [-1, 1), gaussian fp32 with an
    odd count and an odd start position (pairs relative to the start)."""
    from oracle.cpu_baseline import CpuPath

    c = CpuPath(workers=3)
    try:
        key = O.seed_philox(777)
        n = 3 * 4096 + 5
        u = c.burn_philox_uniform(key, 7, n)
        assert np.array_equal(u, O.words_to_unit(O.philox_words(key, 7, n), "fp32"))
        s1, s2 = O.seed_mrg(777)
        m = c.burn_mrg_uniform(s1, s2, 5001, -1.0, 1.0, "fp64")
        assert np.array_equal(m, O.range_transform(O.words_to_unit(O.mrg_fill(*s1, *s2, 5001)[0], "fp64"), -1.0, 1.0))
        g = c.burn_philox_gaussian(key, 3, n)
        words = O.philox_words(key, 3, n + 1)
        assert np.array_equal(g, O.gaussian_from_words(words, 0.0, 1.0, n, "fp32"))
    finally:
        c.close()
