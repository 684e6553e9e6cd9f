"""PCIe copy bandwidth probe (dev tool): D2H / H2D pinned, one vs two streams, concurrent."""
import torch, time
dev = torch.device("cuda", 0)
n = 1 << 30
d = torch.empty(n, dtype=torch.uint8, device=dev)
d2 = torch.empty(n, dtype=torch.uint8, device=dev)
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
def d2h(): h.copy_(d, non_blocking=True)
def h2d(): d.copy_(h, non_blocking=True)
def d2h_two():
    with torch.cuda.stream(s1): h[: n // 2].copy_(d[: n // 2], non_blocking=True)
    with torch.cuda.stream(s2): h[n // 2:].copy_(d[n // 2:], non_blocking=True)
def both():
    with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
for name, fn, b in [("d2h", d2h, n), ("h2d", h2d, n), ("d2h 2 streams", d2h_two, n), ("d2h + h2d concurrent", both, 2 * n)]:
    dt = t(fn)
    print(f"{name}: {b / dt / 1e9:.1f} GB/s")
