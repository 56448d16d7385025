"""Board power and SM clock while the forward transform (r2c rows + two
column passes) loops alone, against the full pair, 1024^3 float64, p = 1.
Instantaneous NVML power sampled every 10 ms inside each timed loop."""
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml as nv
import torch

import paper_1406_5597_b200 as tf

n = int(os.environ.get("N", "1024"))
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)


def sample(stop, out):
    while not stop.is_set():
        fv = nv.nvmlDeviceGetFieldValues(h, [nv.NVML_FI_DEV_POWER_INSTANT])[0]
        out.append((fv.value.uiVal / 1000.0, nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
        stop.wait(0.01)


grid = tf.GlobalGrid(n, n, n)
fp = tf.plan(grid, tf.make_communicators(1)[0], check_consistency=False)
x = torch.rand(n * n * n, dtype=torch.float64, device="cuda") * 2 - 1
slab = tf.RealSlab(fp.real_layout, x)


def run(name, fn, iters):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    time.sleep(1.0)  # let the board cool to the same starting point
    out, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(stop, out))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    th.start()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    while not e1.query():
        time.sleep(0.002)
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / iters
    loaded = out[len(out) // 4:]  # skip the ramp
    w = statistics.median(s[0] for s in loaded)
    mhz = statistics.median(s[1] for s in loaded)
    print(f"{name:28s} {ms:8.3f} ms  median {w:7.1f} W  SM {mhz:6.0f} MHz  {w * ms:9.1f} mJ per call")


run("forward (r2c + 2 columns)", lambda: tf.forward(fp, slab), 60)
run("pair (forward + inverse)", lambda: tf.inverse(fp, tf.forward(fp, slab)), 30)
run("forward (r2c + 2 columns)", lambda: tf.forward(fp, slab), 60)
