"""Stage-1 time per plane with the slab L2-resident (few planes) vs streamed from HBM."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1406_5597_b200 as tf

ep = tf.make_communicators(1)[0]
for dtype, n0s in (("float64", (2, 4, 1024)), ("float32", (4, 8, 1024))):
    for n0 in n0s:
        grid = tf.GlobalGrid(n0, 1024, 1024)
        fp = tf.plan(grid, ep, check_consistency=False, dtype=dtype)
        x = (torch.rand(n0 * 1024 * 1024, dtype=torch.float64, device="cuda") * 2 - 1).to(tf.DTYPES[dtype][1])
        slab = tf.RealSlab(fp.real_layout, x)
        for _ in range(3):
            tf.inverse(fp, tf.forward(fp, slab))
        torch.cuda.synchronize()
        fp.enable_timing(); fp.reset_instrumentation()
        it = max(3, 4096 // n0)
        for _ in range(it):
            tf.inverse(fp, tf.forward(fp, slab))
        t = fp.timers_us
        print(f"{dtype} n0={n0}: stage1+1' per plane {t['stage1_us'] / it / n0:.2f} us, stage3+3' per plane {t['stage3_us'] / it / n0:.2f} us")
        fp.close()
