#!/usr/bin/env python3
"""Per-launch time series of back-to-back headline launches (unit fp32, 2^32),
with nvidia-smi clocks/power sampled alongside: is the launch-to-launch
spread thermal/power drift or noise?  tools/launch_series.py [log2n] [launches]"""
import subprocess
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2109_01329_b200 as P

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 32
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 200
n = 1 << lg
out = torch.empty(n, dtype=torch.float32, device="cuda")
st = P.seed_engine(P.EngineKind.PHILOX4X32X10, 777)
spec = P.Uniform(0.0, 1.0)
for _ in range(3):
    P.generate(spec, st, n, out=out)
torch.cuda.synchronize()
samples, stop = [], threading.Event()


def smi():
    while not stop.is_set():
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,"
                            "clocks_throttle_reasons.active", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True).stdout.strip()
        samples.append((time.time(), r))
        time.sleep(0.05)


th = threading.Thread(target=smi)
th.start()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nl)]
t0 = time.time()
for a, b in ev:
    a.record()
    P.generate(spec, st, n, out=out)
    b.record()
torch.cuda.synchronize()
stop.set()
th.join()
ms = [a.elapsed_time(b) for a, b in ev]
for i in range(0, nl, max(1, nl // 25)):
    chunk = ms[i:i + max(1, nl // 25)]
    print(f"launch {i:4d}-{i + len(chunk) - 1:4d}: mean {sum(chunk) / len(chunk):.4f} ms  min {min(chunk):.4f}  max {max(chunk):.4f}")
print("overall min %.4f median %.4f max %.4f" % (min(ms), sorted(ms)[nl // 2], max(ms)))
for t, r in samples[:: max(1, len(samples) // 20)]:
    print(f"t+{t - t0:6.3f}s smi: {r}")
