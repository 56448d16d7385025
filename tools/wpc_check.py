"""Warp-per-column kernel (TFFFT_WPC=1) against the default TMA column kernel: bitwise, p = 1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1406_5597_b200 as tf

CASES = [((1024, 16, 8), "float64"), ((8, 1024, 16), "float64"), ((1024, 1024, 4), "float64"),
         ((1024, 1024, 32), "float64"), ((1024, 16, 8), "float32"), ((1024, 1024, 64), "float32"), ((16, 1024, 1024), "float64")]
bad = 0
for shape, dtype in CASES:
    x = oracle.uniform_field(shape, seed=5)
    if dtype == "float32":
        x = x.astype(np.float32).astype(np.float64)
    grid = tf.GlobalGrid(*shape)
    ep = tf.make_communicators(1)[0]
    slab = tf.scatter_real(x, grid, 1, dtype=dtype)[0]
    out = {}
    for mode in ("0", "1"):
        os.environ["TFFFT_WPC"] = mode
        fp = tf.plan(grid, ep, dtype=dtype)
        for rep in range(3):
            spec = tf.forward(fp, slab).data.clone()
            back = tf.inverse(fp, tf.SpectralSlab(fp.spectral_layout, tf.SpectralTag.STRIDED_INPLACE, spec.clone())).data.clone()
        torch.cuda.synchronize()
        out[mode] = (spec.cpu().numpy(), back.cpu().numpy(), fp.counters.snapshot())
        fp.close()
    same = np.array_equal(out["0"][0], out["1"][0]) and np.array_equal(out["0"][1], out["1"][1])
    ref = oracle.forward_all(x, 1)[0]
    err = np.linalg.norm(out["1"][0] - ref) / np.linalg.norm(ref)
    rt = np.linalg.norm(out["1"][1] - x.reshape(-1)) / np.linalg.norm(x)
    print(shape, dtype, "bitwise", same, "rel vs oracle %.2e" % err, "round trip %.2e" % rt, flush=True)
    bad += not same
print("FAILED" if bad else "ALL OK")
sys.exit(1 if bad else 0)
