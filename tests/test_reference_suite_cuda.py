"""The reference's OWN test suite through the CUDA plugin seam (needs a GPU).

baseline/stage_ref.sh stages /root/reference/pkg into baseline/_ref/pkg
(git-ignored; it travels to the GPU box), builds its Cython core, adds the
INTEGRATION.md ctypes stub as portarng/_kernels/_cuda.py and patches the
staged selector (_kernels/__init__.py:10-27) to accept
PORTARNG_KERNELS=cuda.  With that selection every caller above the seam --
engine.generate_words, distributions.fill_uniform_unit / fill_gaussian,
rngburn.burn_once, calosim -- draws its words and Box-Muller pairs from
libprng_b200.so on the B200, and the reference's unchanged tests
(test_engine, test_distributions, test_rngburn, test_calosim, test_execution,
test_metrics, test_acceptance) must pass.  test_kernels_cuda.py is the
reference's test_kernels.py with its compiled-core slot bound to the CUDA
module (bitwise words vs the numpy fallback, the 128-bit carry, MRG windows,
box_muller to rtol = atol = 1e-13).

The one expected failure is test_kernels.py::test_an_implementation_is_selected,
which asserts IMPL in ("core", "fallback"); with the plugin selected IMPL is
"cuda".
"""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

REPO = Path(__file__).resolve().parent.parent
STAGED = REPO / "baseline" / "_ref" / "pkg"
LIB = REPO / "paper_2109_01329_b200" / "libprng_b200.so"
EXPECTED_FAILURES = {"tests/test_kernels.py::test_an_implementation_is_selected"}

if not (STAGED / "tests").is_dir():  # pragma: no cover
    pytest.skip("baseline/_ref not staged (run baseline/stage_ref.sh where /root/reference exists)",
                allow_module_level=True)


def run_suite(extra=()):
    env = dict(os.environ, PORTARNG_KERNELS="cuda", PRNG_B200_LIB=str(LIB), PYTHONPATH=str(STAGED / "src"))
    r = subprocess.run([sys.executable, "-m", "pytest", "tests", "-q", "-rfE", "-p", "no:cacheprovider", *extra],
                       cwd=STAGED, env=env, capture_output=True, text=True, timeout=1800)
    return r


def test_reference_suite_passes_with_the_cuda_plugin():
    r = run_suite()
    out = r.stdout + r.stderr
    failed = set(re.findall(r"^(?:FAILED|ERROR) (\S+?)(?: - .*)?$", out, re.M))
    summary = [line for line in out.splitlines() if re.search(r"\d+ (passed|failed)", line)]
    (REPO / "gpurun_out").mkdir(exist_ok=True)
    (REPO / "gpurun_out" / "reference_suite_cuda.txt").write_text(out)
    assert failed <= EXPECTED_FAILURES, f"unexpected failures: {sorted(failed - EXPECTED_FAILURES)}\n{out[-4000:]}"
    assert summary and re.search(r"(\d+) passed", summary[-1]) and int(
        re.search(r"(\d+) passed", summary[-1]).group(1)) >= 150, out[-2000:]


def test_selector_really_binds_the_gpu():
    env = dict(os.environ, PORTARNG_KERNELS="cuda", PRNG_B200_LIB=str(LIB), PYTHONPATH=str(STAGED / "src"))
    code = ("import portarng._kernels as k, portarng.engine as e, portarng.distributions as d;"
            "st = e.seed_engine(e.EngineKind.PHILOX4X32X10, 777);"
            "_, b = d.fill_uniform_unit(st, 1 << 24, 'fp32');"
            "import hashlib; print(k.IMPL, hashlib.sha256(b.values.tobytes()).hexdigest()[:16])")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    # C1 fp32 hash of the unmodified reference
    assert r.stdout.split() == ["cuda", "5b6b175910504b73"]
