"""PCIe copy bandwidth: H2D, D2H, and both directions concurrently (pinned)."""
import time
import torch

n = 8 * 1024 ** 3 // 8  # 8 GiB of float64
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in [("h2d", lambda: d_a.copy_(h_in, non_blocking=True)),
                 ("d2h", lambda: h_out.copy_(d_b, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); fn(); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"{name}: {8 / dt:.1f} GiB/s")
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s1):
    d_a.copy_(h_in, non_blocking=True)
with torch.cuda.stream(s2):
    h_out.copy_(d_b, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t
print(f"both directions concurrently: {16 / dt:.1f} GiB/s total ({dt * 1e3:.0f} ms for 8+8 GiB)")
