import time, torch
n = 38204996 + 1000
for it in range(6):
    t0 = time.perf_counter()
    a = torch.empty(n, dtype=torch.int32, pin_memory=True)
    b = torch.empty(n, dtype=torch.float64, pin_memory=True)
    t1 = time.perf_counter()
    a.fill_(1); b.fill_(1)
    del a, b
    print(f"iter {it}: pinned alloc {1e3*(t1-t0):.2f} ms")
x = torch.empty(1 << 20, device="cuda")
for it in range(4):
    t0 = time.perf_counter()
    a = torch.empty(n, dtype=torch.int32, pin_memory=True)
    b = torch.empty(n, dtype=torch.float64, pin_memory=True)
    a.copy_(x[:1000].int().repeat(n // 1000 + 1)[:n].cpu(), non_blocking=False)
    t1 = time.perf_counter()
    print(f"iter {it}: pinned alloc (+copy) {1e3*(t1-t0):.2f} ms")
    del a, b
