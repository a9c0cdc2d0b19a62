"""Boundary robustness on the GPU: device restore, plugin drop-in semantics,
capture safety of the exact method, stateful engines through the host path,
the lognormal subnormal range.  Everything goes through the C ABI."""

import json
import os
import subprocess
import sys
import textwrap
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2109_01329_b200 as P  # noqa: E402
from paper_2109_01329_b200 import _kernels as K  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tolerances import check_close, lognormal_allowed  # noqa: E402

REPO = Path(__file__).resolve().parent.parent
PHILOX = P.EngineKind.PHILOX4X32X10


def run_py(code, timeout=300):
    env = dict(os.environ, PYTHONPATH=f"{REPO}:{REPO / 'tests'}")
    r = subprocess.run([sys.executable, "-c", textwrap.dedent(code)], cwd=REPO, env=env, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout + r.stderr
    return r.stdout


def test_current_device_is_restored_after_every_entry_point():
    torch.cuda.set_device(0)
    st = P.seed_engine(PHILOX, 777)
    for spec in (P.UniformBits(), P.Uniform(0.0, 1.0), P.Gaussian(0.0, 1.0), P.Lognormal(0.0, 1.0)):
        P.generate(spec, st, 1000)
        assert torch.cuda.current_device() == 0
    if torch.cuda.device_count() < 2:
        pytest.skip("a second GPU is needed to observe a device switch")
    out = torch.empty(4096, dtype=torch.float32, device="cuda:1")
    P.generate(P.Uniform(0.0, 1.0), st, 4096, out=out)
    assert torch.cuda.current_device() == 0
    assert torch.empty(1, device="cuda").device.index == 0
    want = O.words_to_unit(O.philox_words(O.seed_philox(777), 0, 4096), "fp32")
    assert np.array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("offset", [4, 5, 7, 100])
def test_philox_fill_offset_at_least_4_skips_the_first_block(offset):
    # _core.pyx:49-62: lane = offset >= 4 emits nothing from block b, then
    # continues at block b + 1, word 0
    got = K.philox_fill(777, 0, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0, offset, 37)
    want = O.philox_words((777, 0), ((1 << 96) - 1 + 1) * 4, 37)
    assert np.array_equal(got, want)
    ref = O.ref_core()
    if ref is not None:
        assert np.array_equal(got, ref.philox_fill(777, 0, 0xFFFFFFFF, 0xFFFFFFFF, 0xFFFFFFFF, 0, offset, 37))


@pytest.mark.parametrize("n", [(1 << 24) - 3, (1 << 25) + 12345, 3 * (1 << 24)])
def test_plugin_pipeline_chunks(n):
    got = K.philox_fill(777, 0, 5, 0, 0, 0, 2, n)
    want = O.philox_words((777, 0), 5 * 4 + 2, n)
    assert np.array_equal(got, want)
    words, s1, s2 = K.mrg_fill(777, 777, 777, 777, 777, 777, min(n, (1 << 24) + 7))
    w2, t1, t2 = O.mrg_fill(777, 777, 777, 777, 777, 777, min(n, (1 << 24) + 7))
    assert np.array_equal(words, w2) and tuple(s1) == tuple(t1) and tuple(s2) == tuple(t2)


def test_exact_method_first_call_inside_graph_capture():
    # fresh process: the correction tables do not exist yet when the capture starts
    out = run_py("""
        import numpy as np, torch
        import paper_2109_01329_b200 as P
        from oracle import oracle as O
        st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
        out = torch.empty(8192, dtype=torch.float32, device="cuda")
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            P.generate(P.Gaussian(0.0, 1.0, "fp32", "exact"), st, 8192, out=out)
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        want = O.generate("philox", (O.seed_philox(777), 0), "gaussian", 8192, "fp32", 0.0, 1.0)
        assert np.array_equal(out.cpu().numpy(), want)
        print("ok")
    """)
    assert "ok" in out


@pytest.mark.parametrize("strategy", ["pipelined", "zero_copy"])
def test_host_generator_advances_stateful_engines(strategy):
    from paper_2109_01329_b200.hostpath import HostGenerator

    eng = P.Philox4x32x10(777)
    hg = HostGenerator(strategy=strategy, chunk=1 << 16)
    host = torch.empty(100_003, dtype=torch.float32, pin_memory=True)
    ret = hg.generate(P.Uniform(0.0, 1.0), eng, 100_003, host)
    hg.synchronize()
    assert ret is eng and eng.position == 100_003
    want = O.words_to_unit(O.philox_words(O.seed_philox(777), 0, 100_003), "fp32")
    assert np.array_equal(host.numpy(), want)
    hg.generate(P.UniformBits(), eng, 10, torch.empty(10, dtype=torch.uint32, pin_memory=True))
    hg.synchronize()
    assert eng.position == 100_013
    m = P.Mrg32k3a(777)
    hostm = torch.empty(5000, dtype=torch.float64, pin_memory=True)
    hg.generate(P.Uniform(-1.0, 1.0, "fp64"), m, 5000, hostm)
    hg.synchronize()
    s1, s2 = O.seed_mrg(777)
    want = O.range_transform(O.words_to_unit(O.mrg_fill(*s1, *s2, 5000)[0], "fp64"), -1.0, 1.0)
    assert np.array_equal(hostm.numpy(), want)
    assert m.state == P.skip_ahead(P.seed_engine(P.EngineKind.MRG32K3A, 777), 5000)


def test_shard_state_accepts_engine_objects():
    from paper_2109_01329_b200.sharding import generate_shard, strong_shard

    eng = P.Philox4x32x10(777)
    parts = [generate_shard(P.Uniform(0.0, 1.0), eng, strong_shard(10_000, r, 3)).cpu().numpy() for r in range(3)]
    assert eng.position == 0
    want = O.words_to_unit(O.philox_words(O.seed_philox(777), 0, 10_000), "fp32")
    assert np.array_equal(np.concatenate(parts), want)


@pytest.mark.parametrize("m,s", [(-100.0, 1.0), (-80.0, 2.0), (-20.0, 12.0)])
def test_lognormal_fp32_keeps_subnormal_results(m, s):
    st = P.seed_engine(PHILOX, 777)
    n = 1 << 18
    _, x = P.generate(P.Lognormal(m, s, 0.0, 1.0, "fp32"), st, n)
    want = O.generate("philox", (O.seed_philox(777), 0), "lognormal", n, "fp32", m, s)
    got = x.cpu().numpy()
    if m == -100.0:
        # every value is subnormal or underflows to 0 in fp32; most are subnormal
        assert (want < np.finfo(np.float32).tiny).all() and (want > 0).mean() > 0.9
    # m - 5.78 s < -87: the library routes the request to the accurate path (1 ulp)
    check_close(got, want, lognormal_allowed(want, m, s, np.float32, False), "lognormal subnormal range")
    assert np.array_equal(got == 0, want == 0)


def test_write_probe_reports_written_bytes():
    out = torch.empty(1 << 20, dtype=torch.int32, device="cuda")
    P._lib.check(P._lib.lib.prng_diag_write_probe(out.data_ptr(), 4 << 20, None))
    got = out.view(-1, 16).cpu().numpy().astype(np.int64)
    g = np.arange(got.shape[0], dtype=np.int64)[:, None]
    assert np.array_equal(got, g + np.arange(16)[None, :])
    with pytest.raises(P.InvalidParameter):
        P._lib.check(P._lib.lib.prng_diag_write_probe(out.data_ptr() + 4, 64, None))


def test_bench_gpus_2_launches_two_ranks_and_checks_slices():
    # on a 1-GPU box this is the shared-GPU dry run (gloo); on a multi-GPU
    # box it is the real NCCL launch
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--workload", "c1", "--steps", "3",
                        "--warmup", "3", "--no-e2e", "--no-cpu", "--sustained", "0"], cwd=REPO,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["slice_check"]["all_equal"] and line["slice_check"]["ranks"] == 2
    assert len(line["ranks"]) == 2
    if torch.cuda.device_count() >= 2:
        assert line["backend"] == "nccl" and not line["config"]["shared_gpu_dry_run"]
        assert len({x["uuid"] for x in line["ranks"]}) == 2
