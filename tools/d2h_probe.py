import torch, time
n = 1 << 30
d = torch.empty(n, dtype=torch.float32, device="cuda")
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
for chunk in (1 << 22, 1 << 24, 1 << 25, 1 << 26, 1 << 28, n):
    torch.cuda.synchronize()
    ts = []
    for rep in range(3):
        t = time.perf_counter()
        for s in range(0, n, chunk):
            h[s:s + chunk].copy_(d[s:s + chunk], non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    print(f"D2H chunk 2^{chunk.bit_length()-1}: {4 * n / min(ts) / 1e9:.1f} GB/s")
s2 = [torch.cuda.Stream() for _ in range(2)]
torch.cuda.synchronize()
t = time.perf_counter()
chunk = 1 << 25
for i, s in enumerate(range(0, n, chunk)):
    with torch.cuda.stream(s2[i % 2]):
        h[s:s + chunk].copy_(d[s:s + chunk], non_blocking=True)
torch.cuda.synchronize()
print(f"D2H 2 streams chunk 2^25: {4 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
