"""Exact Box-Muller method (PRNG_METHOD_EXACT): pinned to the reference.

CPU: the host tables the library tabulates from libm reproduce the
reference's compiled core (_core.box_muller, oracle/_ref) on EVERY point of
their domains -- all 2^24 u1' with all 2^24 u2 (paired i <-> i), and all 2^24
u1' with u2 = 0 (z0 = r exactly) -- so r*cos/r*sin from the tables equal the
core's outputs bit for bit.  GPU: generate(..., method="exact") equals the
reference's gaussian golden vectors and the oracle exactly, fp32 and fp64,
Philox and MRG, odd n and odd start positions."""

import numpy as np
import pytest

import paper_2109_01329_b200 as P
from oracle import oracle as O
from paper_2109_01329_b200 import distributions as D

N24 = 1 << 24


@pytest.fixture(scope="module")
def tables():
    return D.exact_tables_host()


def test_exact_tables_reproduce_reference_core_on_whole_domain(tables):
    core = O.ref_core()
    if core is None:
        pytest.skip("oracle/_ref not built (oracle/build_ref.sh)")
    log_tab, sc_tab = tables
    u1p = np.arange(1, N24 + 1, dtype=np.float64) * 2.0 ** -24  # 1 - u1 for every 24-bit u1
    u2 = np.arange(N24, dtype=np.float64) * 2.0 ** -24
    r = np.sqrt(-2.0 * log_tab)
    z0, z1 = core.box_muller(u1p, u2)
    assert np.array_equal(z0.view(np.uint64), (r * sc_tab[:, 1]).view(np.uint64))
    assert np.array_equal(z1.view(np.uint64), (r * sc_tab[:, 0]).view(np.uint64))
    z0, _ = core.box_muller(u1p, np.zeros(N24))
    assert np.array_equal(z0.view(np.uint64), r.view(np.uint64))  # cos(0) = 1: z0 = r


def test_exact_method_validation():
    P.Gaussian(0.0, 1.0, "fp64", "exact")
    with pytest.raises(P.InvalidParameter):
        P.Lognormal(method="exact")  # exact is gaussian-only (exp has no finite domain)
    with pytest.raises(P.InvalidParameter):
        P.Gaussian(0.0, 1.0, method="exactish")


torch = pytest.importorskip("torch")


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="no CUDA device")
@pytest.mark.parametrize("engine", ["philox", "mrg"])
@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_exact_gaussian_bit_identical_to_oracle(engine, prec):
    kind = P.EngineKind.PHILOX4X32X10 if engine == "philox" else P.EngineKind.MRG32K3A
    for seed, skip, n, mean, sd in ((777, 0, 1 << 20, 0.0, 1.0), (5, 3, 100001, 2.0, 0.5),
                                    (9, 1, 7, -1.5, 3.25), (11, 0, 1, 0.0, 1.0)):
        st = P.seed_engine(kind, seed)
        st = P.skip_ahead(st, skip) if skip else st
        _, got = P.generate(P.Gaussian(mean, sd, prec, "exact"), st, n)
        ost = (O.seed_philox(seed), skip) if engine == "philox" else O.mrg_skip(*O.seed_mrg(seed), skip)
        want = O.generate(engine, ost, "gaussian", n, prec, mean, sd)
        g = got.cpu().numpy()
        assert g.dtype == want.dtype
        assert np.array_equal(g.view(np.uint32 if prec == "fp32" else np.uint64),
                              want.view(np.uint32 if prec == "fp32" else np.uint64)), (engine, prec, seed, n)


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="no CUDA device")
def test_exact_gaussian_matches_reference_golden(golden, golden_arrays):
    st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
    _, z = P.generate(P.Gaussian(0.0, 1.0, "fp32", "exact"), st, 1 << 20)
    assert O.sha16(z.cpu().numpy()) == "1d550a2766efec00"  # SURVEY Appendix A, reference core
    words = P.generate_words(st, 4096)[1]
    for prec in ("fp32", "fp64"):
        a = P.gaussian_from_words(words, 0.25, 2.0, 4095, prec, method="exact").cpu().numpy()
        b = O.gaussian_from_words(words.cpu().numpy(), 0.25, 2.0, 4095, prec)
        assert np.array_equal(a, b)


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available(), reason="no CUDA device")
def test_exact_route_rounding_test_bounds_and_cancellation_cases():
    """The fp32 exact route skips the correction tables unless the fp64
    value sits within its error bound of an fp32 rounding boundary.  The
    bounds it uses are the worst approximation errors measured over the
    whole domains; they must be tiny (the short fp64 forms: ~2^-44).  Outputs stay
    bit-identical where the affine cancels (mean ~ -z * sd), the case the
    bound's |v| terms exist for."""
    import ctypes
    import json

    b = (ctypes.c_double * 2)()
    esc = ctypes.c_uint64()
    P._lib.check(P._lib.lib.prng_exact_tables_bounds(b, ctypes.byref(esc)))
    print(json.dumps({"exact_bounds": {"rel_log": b[0], "abs_sincos": b[1], "escapes": esc.value}}))
    assert 0 <= b[0] < 2.0 ** -40 and 0 <= b[1] < 2.0 ** -40
    st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 2024)
    for mean, sd in ((-1.0, 1.0), (1.0, 1.0), (1e-3, 1e-3), (-3.0, 1.0), (0.0, 1e-30), (1e20, 1e20)):
        n = 1 << 20
        _, got = P.generate(P.Gaussian(mean, sd, "fp32", "exact"), st, n)
        want = O.generate("philox", (O.seed_philox(2024), 0), "gaussian", n, "fp32", mean, sd)
        assert np.array_equal(got.cpu().numpy().view(np.uint32), want.view(np.uint32)), (mean, sd)

