"""Property-based and statistical checks on the device path (reference test
strategy: hypothesis random (key, counter) vs the oracle,
test_engine.py:31-37; uniform mean / chi^2 band and normal mean/std,
test_distributions.py:68-71, 135-140, 170-179)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

import paper_2109_01329_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

U32 = st.integers(0, 2**32 - 1)


@settings(max_examples=120, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(k0=U32, k1=U32, c=st.tuples(U32, U32, U32, U32), lane=st.integers(0, 3), n=st.integers(0, 5000),
       dist=st.sampled_from(["bits", "uniform32", "uniform64", "gauss_exact32", "gauss_exact64"]),
       lo=st.floats(-1e6, 1e6, allow_nan=False), width=st.floats(1e-3, 1e6))
def test_random_philox_requests_equal_oracle(k0, k1, c, lane, n, dist, lo, width):
    state = P.PhiloxState((k0, k1), c, lane_index=4)
    state = P.skip_ahead(state, lane) if lane else state
    pos = P.stream_position(state)
    key = (k0, k1)
    if dist == "bits":
        got = P.generate(P.UniformBits(), state, n)[1].cpu().numpy()
        want = O.philox_words(key, pos, n)
    elif dist.startswith("uniform"):
        prec = "fp32" if dist.endswith("32") else "fp64"
        got = P.generate(P.Uniform(lo, lo + width, prec), state, n)[1].cpu().numpy()
        want = O.generate("philox", (key, pos), "uniform", n, prec, lo, lo + width)
    else:
        prec = "fp32" if dist.endswith("32") else "fp64"
        got = P.generate(P.Gaussian(lo, width, prec, "exact"), state, n)[1].cpu().numpy()
        want = O.generate("philox", (key, pos), "gaussian", n, prec, lo, width)
    assert got.dtype == want.dtype and np.array_equal(got, want, equal_nan=True)


@settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(seed=st.integers(0, 2**64 - 1), skip=st.integers(0, 2**40), n=st.integers(0, 30000))
def test_random_mrg_requests_equal_oracle(seed, skip, n):
    state = P.skip_ahead(P.seed_engine(P.EngineKind.MRG32K3A, seed), skip)
    s1, s2 = O.mrg_skip(*O.seed_mrg(seed), skip)
    got = P.generate(P.UniformBits(), state, n)[1].cpu().numpy()
    assert np.array_equal(got, O.mrg_fill(*s1, *s2, n)[0])


@pytest.mark.parametrize("engine", [P.EngineKind.PHILOX4X32X10, P.EngineKind.MRG32K3A])
def test_statistics(engine):
    n = 1 << 24
    st0 = P.seed_engine(engine, 2024)
    u = P.generate(P.Uniform(0.0, 1.0), st0, n)[1]
    assert abs(float(u.double().mean()) - 0.5) < 0.002
    counts = torch.histc(u, bins=100, min=0.0, max=1.0).double().cpu().numpy()
    chi2 = float(((counts - n / 100) ** 2 / (n / 100)).sum())
    assert 50 < chi2 < 160  # chi^2(99): far outside only for a broken generator
    for method in ("fast", "accurate", "exact"):
        z = P.generate(P.Gaussian(0.0, 1.0, "fp32", method), st0, n)[1].double()
        assert abs(float(z.mean())) < 0.005 and abs(float(z.std()) - 1.0) < 0.005, method
    x = P.generate(P.Lognormal(0.0, 0.5, 0.0, 1.0), st0, n)[1].double()
    assert abs(float(x.mean()) - np.exp(0.125)) < 0.01  # E = exp(m + s^2/2)
