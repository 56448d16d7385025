"""Reference point only (not part of the product): cuFFT via torch.fft on the
same forward+inverse pair, device-timed."""
import sys
import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dt = torch.float64 if (len(sys.argv) < 3 or sys.argv[2] == "float64") else torch.float32
x = (torch.rand(n, n, n, dtype=dt, device="cuda") * 2 - 1)
for _ in range(2):
    y = torch.fft.irfftn(torch.fft.rfftn(x), s=x.shape)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    y = torch.fft.irfftn(torch.fft.rfftn(x), s=x.shape)
e1.record()
torch.cuda.synchronize()
print(f"cuFFT (torch.fft) {n}^3 {dt}: pair {e0.elapsed_time(e1) / 3:.3f} ms, rel err {(y - x).norm().item() / x.norm().item():.2e}")
