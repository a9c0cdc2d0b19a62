"""The stated tolerances live with the oracle (oracle/tolerances.py) so that
bench.py's per-rank slice check can use them without importing tests/."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.tolerances import *  # noqa: E402,F401,F403
from oracle.tolerances import check_close, gaussian_allowed, lognormal_allowed, ulp  # noqa: E402,F401
