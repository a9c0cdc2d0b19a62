import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import torch
import paper_2109_01329_b200 as P
st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
out = torch.empty(1024, device="cuda")
spec = P.Uniform(0.0, 1.0)
for _ in range(1000): P.generate(spec, st, 1024, out=out)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(20000): P.generate(spec, st, 1024, out=out)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
