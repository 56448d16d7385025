"""PCIe copy bandwidth from pinned host memory: H2D, D2H, both directions at
once, and each direction split over k streams (copy engines)."""
import time
import torch

GiB = 1024 ** 3
n = 8 * GiB // 8  # 8 GiB of float64
h_in = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")


def timed(fn):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter(); fn(); torch.cuda.synchronize()
    return time.perf_counter() - t


def split(k, up, down):
    streams = [torch.cuda.Stream() for _ in range(2 * k)]
    c = n // k

    def run():
        for i in range(k):
            if up:
                with torch.cuda.stream(streams[i]):
                    d_a[i * c:(i + 1) * c].copy_(h_in[i * c:(i + 1) * c], non_blocking=True)
            if down:
                with torch.cuda.stream(streams[k + i]):
                    h_out[i * c:(i + 1) * c].copy_(d_b[i * c:(i + 1) * c], non_blocking=True)
    return run


for k in (1, 2, 4):
    for up, down, name in ((True, False, "h2d"), (False, True, "d2h"), (True, True, "both")):
        dt = timed(split(k, up, down))
        gib = 8 * (up + down)
        print(f"{name:5s} streams/dir={k}: {gib / dt:6.1f} GiB/s ({dt * 1e3:.0f} ms for {gib} GiB)")
