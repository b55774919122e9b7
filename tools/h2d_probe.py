"""H2D/D2H bandwidth from pageable numpy vs pinned host memory (e2e staging design)."""
import time, numpy as np, torch
n = 158_000_000
h = np.random.default_rng(0).integers(0, 255, n, dtype=np.uint8)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
p = torch.empty(n, dtype=torch.uint8).pin_memory()
p.numpy()[:] = h
for name, src in (("pageable", torch.from_numpy(h)), ("pinned", p)):
    for _ in range(2):
        d.copy_(src); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        d.copy_(src, non_blocking=True); torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print("H2D %s: %.2f ms (%.1f GB/s)" % (name, dt * 1e3, n / dt / 1e9))
t = time.perf_counter()
for _ in range(5):
    np.copyto(p.numpy(), h)
dt = (time.perf_counter() - t) / 5
print("host memcpy 1 thread into pinned: %.2f ms (%.1f GB/s)" % (dt * 1e3, n / dt / 1e9))
import os; print("cpus", os.cpu_count())
