#!/usr/bin/env python3
"""Small requests through every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): tools/sanitize.sh."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2109_01329_b200 as P
from paper_2109_01329_b200 import calosim as C
from paper_2109_01329_b200 import execution as X

ph = P.skip_ahead(P.seed_engine(P.EngineKind.PHILOX4X32X10, 5), 3)
mr = P.seed_engine(P.EngineKind.MRG32K3A, 5)
for st in (ph, mr):
    for spec in (P.UniformBits(), P.UniformBits(64), P.Uniform(-1.0, 2.0), P.Uniform(0.0, 1.0, "fp64"),
                 P.Gaussian(0.0, 1.0), P.Gaussian(0.0, 1.0, "fp64"), P.Gaussian(1.0, 2.0, "fp32", "exact"),
                 P.Lognormal(), P.Lognormal(0.1, 0.3, 0.0, 1.0, "fp64")):
        for n in (1, 37, 4099, 100003):
            P.generate(spec, st, n)
# MRG fp64 segmented path with several rounds (per-lane jumps) per chain
P.generate(P.Uniform(-1.0, 2.0, "fp64"), mr, (1 << 25) + 12345)
w = P.generate_words(ph, 1002)[1]
P.gaussian_from_words(w, 0.0, 1.0, 1001)
P.words_to_unit(w, "fp64")
tab = C.segment_table(12345, [100, 0, 5000, 7])
out = torch.empty(6000, device="cuda")
C.generate_segments(ph, tab, out)
geom = [np.arange(r, 1200, 4, dtype=np.int64) for r in range(4)]
det = C.Detector(geom, {"electron": C.Parameterization("electron", 40, 90, np.linspace(0.001, 0.101, 9),
                                                       np.full(8, 0.125))})
ev = C.synth_single_electron_events(20, 777)
C.simulate_events(ev, det, P.seed_engine(P.EngineKind.PHILOX4X32X10, 777), min_batch=500)
# deposit kernel on its own: two windows (ids up to 2^20), > 4096 unique cells, one hot cell
from paper_2109_01329_b200 import _lib
rng = np.random.default_rng(3)
cells = np.concatenate([rng.integers(0, 1 << 20, 6000), np.full(300, 77), rng.integers(0, 64, 50)]).astype(np.int32)
offs = torch.tensor([0, 6000, 6000, 6300, 6350], dtype=torch.int64, device="cuda")
d_c = torch.from_numpy(cells).cuda()
d_a = torch.rand(len(cells), dtype=torch.float64, device="cuda")
nb = _lib.lib.prng_calo_deposit_scratch_bytes(len(cells), 4)
scr = torch.empty(nb, dtype=torch.uint8, device="cuda")
oc = torch.empty(len(cells), dtype=torch.int32, device="cuda")
oe = torch.empty(len(cells), dtype=torch.float64, device="cuda")
oo = torch.empty(5, dtype=torch.int64, device="cuda")
_lib.check(_lib.lib.prng_calo_deposit(d_c.data_ptr(), d_a.data_ptr(), len(cells), offs.data_ptr(), 4, 0, scr.data_ptr(),
                                      nb, oc.data_ptr(), oe.data_ptr(), oo.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream))
g = X.TaskGraph()
b = g.create_buffer(10007)
g.submit_with_accessors(X.uniform_generate_kernel(ph, b.id, "fp32"), [(b, X.AccessMode.READ_WRITE)])
g.submit_with_accessors(X.affine_kernel(b.id, -1.0, 1.0), [(b, X.AccessMode.READ_WRITE)])
g.run(X.Parallel(3, chunk=997))
g.copy_to_host(b)
torch.cuda.synchronize()
print("sanitize target: ok")
