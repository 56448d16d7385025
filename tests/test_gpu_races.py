"""Race and coverage checks of the kernels and the exchange (compute-sanitizer
is closed on this pool, so the invariants are checked by construction).

1. Coverage, "each (src, dst, slot) is written exactly once" (the reference
   fabric's invariant, transport.py:17-19): before every call the plan's
   exchange staging / landing buffers and the output buffers are filled with
   NaN (FftPlan.poison, tensor.fill_).  Any element a stage reads that no
   stage (or peer) wrote -- a missed band, a chunk landing at the wrong
   offset, a consumer running before its producer -- propagates NaN into the
   result, which must instead equal the oracle.
2. Races: shared-memory hand-offs (TMA boxes and mbarriers, the ticket tile
   queue, the split-word exchange), the local-fabric events and the batched
   pipeline's cross-stream hand-offs.  A race shows up as run-to-run
   variation; every case runs 12 times and every run must be BITWISE equal to
   the first.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_1406_5597_b200 as tf

pytestmark = pytest.mark.gpu
REPS = 12

CASES = [
    ((1024, 32, 16), 1, {}),                                             # TMA columns (FPF), n0 = 1024
    ((32, 1024, 16), 1, {"dtype": "float32"}),                           # f32 stage 1b parity maps
    ((1024, 64, 16), 2, {}),                                             # two-level TMA p = 2
    ((512, 64, 32), 4, {"comm_pattern": tf.CommPattern.COLLECTIVE}),
    ((1024, 32, 16), 8, {"algorithms": ("peer_stores", "tma_columns")}),
    ((256, 128, 32), 4, {"algorithms": ()}),                             # cp.async column kernel
    ((64, 64, 32), 4, {"batch": 3}),                                     # batched pipeline, 2 buffer sets
    ((512, 32, 16), 2, {"batch": 4, "algorithms": ("peer_stores", "tma_columns")}),
    ((1024, 32, 16), 4, {"algorithms": ("chunked_exchange", "tma_columns")}),      # plane-chunked forward
    ((16, 1024, 32), 1, {}),                                             # warp-per-column stage 1b, p = 1
    ((32, 1024, 16), 4, {}),                                             # warp-per-column two-level stage 1b
    ((32, 1024, 16), 8, {"algorithms": ("peer_stores", "tma_columns")}),  # ... storing into the peers' landing
    ((32, 1024, 16), 2, {"batch": 3}),                                   # ... in the batched pipeline
    ((2048, 32, 16), 1, {}),                                             # 2 x 1024 tensor-memory kernel, stage 3
    ((16, 2048, 32), 4, {}),                                             # ... two-level stage 1b (5D landing loads)
    ((2048, 32, 16), 2, {"algorithms": ("chunked_exchange", "tma_columns")}),  # ... with the chunked exchange
    ((512, 64, 16), 4, {"algorithms": ("chunked_exchange", "tma_columns")}),   # chunked, both directions, 512 points
]


@pytest.mark.parametrize("shape,p,kw", CASES, ids=lambda v: str(v))
def test_poisoned_repeated_runs_are_exact_and_bitwise_stable(shape, p, kw):
    kw = dict(kw)
    batch = kw.get("batch", 1)
    dtype = kw.get("dtype", "float64")
    tol = 1e-12 if dtype == "float64" else 1e-5
    grid = tf.GlobalGrid(*shape)
    fields = [oracle.uniform_field(shape, seed=90 + c) for c in range(batch)]
    if dtype == "float32":
        fields = [f.astype(np.float32).astype(np.float64) for f in fields]
    slabs = [tf.scatter_real(x, grid, p, dtype=dtype) for x in fields]

    def body(ep):
        fp = tf.plan(grid, ep, tf.Strategy.STRIDED, **kw)
        real = torch.cat([slabs[c][ep.rank].data for c in range(batch)])
        outs = []
        for _ in range(REPS):
            ep.barrier()
            fp.poison()
            fp.work1.fill_(float("nan"))
            fp.real_out.fill_(float("nan"))
            ep.barrier()
            if batch > 1:
                spec = tf.forward_many(fp, real)
                s = spec.clone()
                back = tf.inverse_many(fp, spec)
            else:
                spec = tf.forward(fp, tf.RealSlab(fp.real_layout, real)).data
                s = spec.clone()
                back = tf.inverse(fp, tf.SpectralSlab(fp.spectral_layout, tf.SpectralTag.STRIDED_INPLACE, spec)).data
            outs.append((s.cpu().numpy(), back.clone().cpu().numpy()))
        ep.barrier()
        fp.close()
        return outs

    res = tf.run_spmd(p, body)
    for q in range(p):
        s0, b0 = res[q][0]
        for s, b in res[q][1:]:
            assert np.array_equal(s.view(np.uint8), s0.view(np.uint8)), f"rank {q}: spectra differ between runs"
            assert np.array_equal(b.view(np.uint8), b0.view(np.uint8)), f"rank {q}: inverse outputs differ"
        assert np.all(np.isfinite(s0)) and np.all(np.isfinite(b0)), f"rank {q}: NaN from a poisoned buffer"
    for c in range(batch):
        ref = oracle.forward_all(fields[c], p)
        for q in range(p):
            got = res[q][0][0].reshape(batch, -1)[c]
            assert np.linalg.norm(got - ref[q]) / np.linalg.norm(ref[q]) <= tol
        back = np.concatenate([res[q][0][1].reshape(batch, -1)[c] for q in range(p)]).reshape(shape)
        assert np.linalg.norm(back - fields[c]) / np.linalg.norm(fields[c]) <= tol
