"""Host<->device copy ceiling for the e2e leg of bench.py: pinned 1 GiB
H2D, D2H, and both directions at once on two streams.

    python tools/pcie_probe.py
"""
import torch, time
n = 1 << 27  # 1 GiB fp64
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h2.copy_(d2, non_blocking=True))):
    t = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(name, round(n * 8 / dt / 1e9, 1), "GB/s")
t = time.perf_counter()
with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print("both", round(2 * n * 8 / dt / 1e9, 1), "GB/s aggregate")
