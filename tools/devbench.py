"""Developer timing: forward+inverse pair at one grid, p=1, CUDA events; per-stage times."""
import argparse
import sys
import os
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
if os.environ.get("HUGE_ALLOC"):  # experiment: large buffers through tools/micro/libhugealloc.so (512 MB-aligned VMM mappings)
    _so = os.path.join(os.path.dirname(os.path.abspath(__file__)), "micro", "libhugealloc.so")
    torch.cuda.memory.change_current_allocator(torch.cuda.memory.CUDAPluggableAllocator(_so, "huge_malloc", "huge_free"))
import paper_1406_5597_b200 as tf

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--dtype", default="float64")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--check", action="store_true")
ap.add_argument("--shape", default=None, help="n0,n1,n2 (overrides --n)")
a = ap.parse_args()
n = a.n
n0, n1, n2 = (int(v) for v in a.shape.split(",")) if a.shape else (n, n, n)
grid = tf.GlobalGrid(n0, n1, n2)
ep = tf.make_communicators(1)[0]
fp = tf.plan(grid, ep, check_consistency=False, dtype=a.dtype)
rdt = tf.DTYPES[a.dtype][1]
x = (torch.rand(n0 * n1 * n2, dtype=torch.float64, device="cuda") * 2 - 1).to(rdt)
slab = tf.RealSlab(fp.real_layout, x)
for _ in range(int(os.environ.get("WARM", "2"))):
    tf.inverse(fp, tf.forward(fp, slab))
torch.cuda.synchronize()
fp.enable_timing()
fp.reset_instrumentation()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    tf.inverse(fp, tf.forward(fp, slab))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
N = n0 * n1 * n2
import math
gflops = 5 * N * math.log2(N) / (ms * 1e-3) / 1e9
s_r = 8 if a.dtype == "float64" else 4
hbm = 2 * (s_r * N + 3 * 2 * s_r * n0 * n1 * (n2 // 2 + 1))
t = fp.timers_us
print(f"n={n0}x{n1}x{n2} {a.dtype} pair {ms:.3f} ms  {gflops:.0f} GFLOP/s  roofline-HBM(6539) {hbm/6539e9*1e3:.3f} ms -> frac {hbm/6539e9*1e3/ms:.3f}")
print("per-pair stage ms:", {k: round(v / 1e3 / a.iters, 3) for k, v in t.items()})
if a.check:
    xr = x.double().view(n0, n1, n2)
    ref = torch.fft.rfftn(xr)
    spec = tf.forward(fp, slab).data.view(n0, n1, n2 // 2 + 1).to(torch.complex128)
    err = (torch.linalg.norm(spec - ref) / torch.linalg.norm(ref)).item()
    back = tf.inverse(fp, tf.forward(fp, slab)).data.double()
    rt = (torch.linalg.norm(back - x.double()) / torch.linalg.norm(x.double())).item()
    print(f"check vs torch.fft.rfftn: rel L2 {err:.3e}; round trip {rt:.3e}")
