"""Small-grid runs of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck; one tool per run, B200_PROFILING.md):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Covers: r2c / c2r rows, the TMA column kernel (p = 1 and the two-level p > 1
variant with landing loads and block-table stores), the cp.async column kernel
(persistent ticket queue, RD = 1 / 2 redirects), the local-fabric pull
(PAIRWISE per-peer and COLLECTIVE), peer stores, the batched pipeline, the
opt-in four-step and fused stage 1, and the TRANSPOSE pack / unpack.  Each
case checks its result against the oracle, so a sanitizer-clean run is also a
correct one.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1406_5597_b200 as tf  # noqa: E402

CASES = [
    # shape, p, kwargs for plan
    ((1024, 16, 8), 1, {}),                                      # TMA columns, n0 = 1024 (stage 3)
    ((16, 512, 8), 1, {}),                                       # TMA columns, n1 = 512 (stage 1b)
    ((512, 32, 16), 2, {}),                                      # TMA two-level p = 2
    ((1024, 16, 8), 4, {"comm_pattern": tf.CommPattern.COLLECTIVE}),
    ((1024, 16, 8), 2, {"algorithms": ("peer_stores",)}),
    ((64, 64, 32), 2, {"algorithms": ()}),                       # cp.async column kernel, RD redirects
    ((32, 32, 16), 4, {"batch": 3}),                             # batched pipeline
    ((1024, 8, 16), 1, {"algorithms": ("fourstep_stage3",)}),
    ((8, 1024, 1024), 1, {"algorithms": ("fused_stage1",)}),
    ((16, 16, 16), 2, {"strategy": tf.Strategy.TRANSPOSE}),
]


def run_case(shape, p, kw):
    grid = tf.GlobalGrid(*shape)
    batch = kw.get("batch", 1)
    fields = [oracle.uniform_field(shape, seed=3 + c) for c in range(batch)]
    slabs = [tf.scatter_real(x, grid, p) for x in fields]
    kw = dict(kw)
    strategy = kw.pop("strategy", tf.Strategy.STRIDED)

    def body(ep):
        fp = tf.plan(grid, ep, strategy, **kw)
        if batch > 1:
            real = torch.cat([slabs[c][ep.rank].data for c in range(batch)])
            spec = tf.forward_many(fp, real).clone()
            back = tf.inverse_many(fp, spec.clone()).clone()
        else:
            spec = tf.forward(fp, slabs[0][ep.rank]).data.clone()
            back = tf.inverse(fp, tf.forward(fp, slabs[0][ep.rank])).data.clone()
        torch.cuda.synchronize()
        fp.close()
        return spec.cpu().numpy(), back.cpu().numpy()

    res = tf.run_spmd(p, body)
    worst = 0.0
    for c in range(batch):
        x = fields[c]
        back = np.concatenate([res[q][1].reshape(batch, -1)[c] for q in range(p)]).reshape(shape)
        worst = max(worst, float(np.linalg.norm(back - x) / np.linalg.norm(x)))
        if strategy is tf.Strategy.STRIDED:
            ref = oracle.forward_all(x, p)
            for q in range(p):
                got = res[q][0].reshape(batch, -1)[c]
                worst = max(worst, float(np.linalg.norm(got - ref[q]) / np.linalg.norm(ref[q])))
    return worst


def main():
    torch.cuda.set_device(0)
    bad = 0
    for shape, p, kw in CASES:
        e = run_case(shape, p, kw)
        ok = e <= 1e-12
        bad += not ok
        print(f"{shape} p={p} {kw}: worst rel L2 {e:.2e} {'ok' if ok else 'FAIL'}", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
