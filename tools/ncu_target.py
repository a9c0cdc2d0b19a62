#!/usr/bin/env python3
"""Launch a few kernels of one workload for ncu capture: tools/ncu_target.py WORKLOAD [log2n] [reps]."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2109_01329_b200 as P

W = {
    "unit_f32": ("philox", lambda: P.Uniform(0.0, 1.0), torch.float32),
    "uniform_f32": ("philox", lambda: P.Uniform(-3.0, 5.0), torch.float32),
    "bits": ("philox", lambda: P.UniformBits(), torch.uint32),
    "unit_f64": ("philox", lambda: P.Uniform(0.0, 1.0, "fp64"), torch.float64),
    "gauss_f32": ("philox", lambda: P.Gaussian(0.0, 1.0), torch.float32),
    "gauss_f32_acc": ("philox", lambda: P.Gaussian(0.0, 1.0, method="accurate"), torch.float32),
    "gauss_f32_exact": ("philox", lambda: P.Gaussian(0.0, 1.0, method="exact"), torch.float32),
    "gauss_f32_precise": ("philox", lambda: P.Gaussian(0.0, 1.0, method="precise"), torch.float32),
    "logn_f32_precise": ("philox", lambda: P.Lognormal(method="precise"), torch.float32),
    "gauss_f64_exact": ("philox", lambda: P.Gaussian(0.0, 1.0, "fp64", "exact"), torch.float64),
    "gauss_f64": ("philox", lambda: P.Gaussian(0.0, 1.0, "fp64"), torch.float64),
    "logn_f32": ("philox", lambda: P.Lognormal(), torch.float32),
    "mrg_bits": ("mrg", lambda: P.UniformBits(), torch.uint32),
    "mrg_f64": ("mrg", lambda: P.Uniform(-1.0, 1.0, "fp64"), torch.float64),
    "mrg_f32": ("mrg", lambda: P.Uniform(-1.0, 1.0), torch.float32),
    "fill": (None, None, torch.float32),
}


def main():
    name = sys.argv[1]
    n = 1 << int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 28
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    eng, mk, dt = W[name]
    out = torch.empty(n, dtype=dt, device="cuda")
    if eng is None:
        for _ in range(reps):
            out.fill_(1.0)
    else:
        st = P.seed_engine(P.EngineKind.PHILOX4X32X10 if eng == "philox" else P.EngineKind.MRG32K3A, 777)
        spec = mk()
        for _ in range(reps):
            P.generate(spec, st, n, out=out)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
