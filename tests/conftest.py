import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
for p in (str(REPO), str(REPO / "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running test")
    # Build the CUDA library (nvcc cross-compiles without a GPU) and the CPU
    # checker if a fresh checkout lacks them; the package itself never falls
    # back to anything else.
    import subprocess

    if not (REPO / "paper_2109_01329_b200" / "libprng_b200.so").exists():
        subprocess.run(["make", "-s", "-C", str(REPO / "paper_2109_01329_b200" / "csrc")], check=True)
    if not (REPO / "oracle" / "liboracle.so").exists():
        subprocess.run(["make", "-s", "-C", str(REPO / "oracle")], check=True)


@pytest.fixture(scope="session")
def golden():
    return json.loads((GOLDEN / "golden.json").read_text())


@pytest.fixture(scope="session")
def golden_arrays():
    with np.load(GOLDEN / "cases.npz") as z:
        return {k: z[k] for k in z.files}
