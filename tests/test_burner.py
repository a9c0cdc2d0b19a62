"""RNG burner (rngburn.py analogue): result format on CPU, modes on GPU."""

import numpy as np
import pytest

import paper_2109_01329_b200 as P
from paper_2109_01329_b200 import burner as B
from paper_2109_01329_b200 import execution as X


def test_csv_is_byte_identical_to_reference_writer(golden, tmp_path):
    recs = [B.RunRecord("b200", "buffer", "cuda:148sm", "philox", "uniform:-1:1", 1000, [1500, 1400, 1450]),
            B.RunRecord("b200", "usm", "cuda:148sm", "mrg32k3a", "gaussian:2:0.5", 7, [99])]
    path = tmp_path / "r.csv"
    B.write_records_csv(recs, str(path))
    assert path.read_text() == golden["burner_csv"]
    rows = B.read_rows_csv(str(path))
    assert len(rows) == 4 and rows[0]["tts_ns"] == 1500 and rows[3]["engine"] == "mrg32k3a"


def test_csv_schema_mismatch(tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text("platform,api,backend\nx,y,z\n")
    with pytest.raises(B.SchemaMismatch):
        B.read_rows_csv(str(bad))


def test_config_validation_matches_reference():
    good = dict(engine=P.EngineKind.PHILOX4X32X10, dist=P.Uniform(0.0, 1.0), api_mode="buffer",
                backend=X.Serial(), batches=[1])
    B.BurnConfig(**good)
    for bad in ({"api_mode": "cuda"}, {"batches": []}, {"batches": [0]}, {"iterations": 0}):
        with pytest.raises(X.ConfigError):
            B.BurnConfig(**{**good, **bad})
    assert B.dist_label(P.Uniform(-1.0, 1.0)) == "uniform:-1:1"
    assert B.dist_label(P.Gaussian(2.0, 0.5)) == "gaussian:2:0.5"


@pytest.mark.gpu
def test_modes_are_bit_identical_and_match_reference_burn_once(golden_arrays, tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    PH, MRG = P.EngineKind.PHILOX4X32X10, P.EngineKind.MRG32K3A
    for eng, spec, batch, seed, label in (
        (PH, P.Uniform(-1.0, 1.0), 1000, 99, "philox_uniform_m1p1_1000"),
        (MRG, P.Uniform(-1.0, 1.0), 500, 99, "mrg_uniform_m1p1_500"),
        (PH, P.Uniform(-1.0, 1.0, "fp64"), 777, 13, "philox_uniform_f64_m1p1_777"),
        (PH, P.Gaussian(2.0, 0.5, method="accurate"), 1001, 7, "philox_gauss_2_0.5_1001"),
    ):
        outs = [B.burn_once(eng, spec, mode, backend, batch, seed)[1] for mode in B.API_MODES
                for backend in (X.Serial(), X.Parallel(4, chunk=97), X.Graph(3, chunk=250))]
        assert all(np.array_equal(outs[0], o) for o in outs[1:]), label
        want = golden_arrays[f"burn__{label}"]
        if isinstance(spec, P.Uniform):
            assert np.array_equal(outs[0], want), label
        else:  # accurate fp32 gaussian: fp64 math then one cast
            assert np.max(np.abs(outs[0].astype(np.float64) - want)) <= np.max(np.spacing(np.abs(want)))
    cfg = B.BurnConfig(PH, P.Uniform(-1.0, 1.0), "usm", X.Parallel(2), [10, 1000], iterations=3, seed=1,
                       out_path=str(tmp_path / "g.csv"))
    recs = B.run_burner(cfg)
    assert [r.batch for r in recs] == [10, 1000] and all(t > 0 for r in recs for t in r.samples)
    assert recs[0].backend == "parallel:2"
    assert len(B.read_rows_csv(str(tmp_path / "g.csv"))) == 6
