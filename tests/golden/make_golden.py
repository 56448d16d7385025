"""Generate golden fixtures by running the UNMODIFIED reference ``slabfft``.

Run in the build container only (it reads /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

For every case it drives the reference's public API exactly like its own
test helpers (pkg/tests/helpers.py:12-41): ``scatter_real`` -> ``run_spmd``
-> ``plan(grid, ep, Strategy.STRIDED)`` -> ``forward`` -> ``inverse`` and
stores the seeded input parameters, each rank's STRIDED_INPLACE spectral
buffer (forward output), each rank's inverse output and the residue.  The
committed .npz files are what tests/test_oracle.py pins the oracle against.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# (n0, n1, n2, p, dist, seed)
CASES = [
    (2, 2, 2, 1, "normal", 0),
    (2, 2, 2, 2, "normal", 1),
    (4, 8, 4, 2, "normal", 2),
    (8, 4, 2, 4, "normal", 3),
    (8, 8, 8, 1, "uniform", 4),
    (8, 8, 8, 2, "uniform", 5),
    (16, 16, 16, 4, "normal", 6),
    (16, 8, 32, 8, "uniform", 7),
    (32, 32, 32, 2, "uniform", 8),
    (64, 16, 8, 4, "normal", 9),
    (4, 64, 16, 2, "normal", 10),
]


def field(shape, dist, seed):
    rng = np.random.default_rng(seed)
    if dist == "uniform":
        return rng.uniform(-1.0, 1.0, size=shape)
    return rng.standard_normal(shape)


def run_reference(sf, n0, n1, n2, p, values):
    grid = sf.GlobalGrid(n0, n1, n2)
    slabs = sf.scatter_real(values, grid, p)

    def body(ep):
        fp = sf.plan(grid, ep, sf.Strategy.STRIDED)
        spec = sf.forward(fp, slabs[ep.rank])
        fwd = spec.data.copy()
        out = sf.inverse(fp, spec)
        return fwd, out.data.copy(), fp.last_imag_residue

    res = sf.run_spmd(p, body, sf.CommMode.SERIAL)
    return [r[0] for r in res], [r[1] for r in res], max(r[2] for r in res)


def main() -> int:
    if not os.path.isdir(REF):
        print("reference not present; nothing to do")
        return 0
    sys.path.insert(0, REF)
    import slabfft as sf

    for n0, n1, n2, p, dist, seed in CASES:
        x = field((n0, n1, n2), dist, seed)
        fwd, inv, residue = run_reference(sf, n0, n1, n2, p, x)
        name = f"ref_{n0}x{n1}x{n2}_p{p}.npz"
        np.savez_compressed(
            os.path.join(HERE, name),
            shape=np.array([n0, n1, n2]), p=np.array(p), dist=np.array(dist),
            seed=np.array(seed),
            fwd=np.stack(fwd), inv=np.stack(inv), residue=np.array(residue),
        )
        print("wrote", name)

    # Fig. 3 of the paper / SPEC.md:339, 548: STRIDED exchange, 4x4 with n2c=1, p=2.
    grid = sf.GlobalGrid(4, 4, 1)
    data = np.arange(1, 17, dtype=np.complex128).reshape(4, 4, 1)

    def body(ep):
        xp = sf.plan_exchange(grid, 2, ep.rank, sf.Strategy.STRIDED)
        buf = data[ep.rank * 2 : (ep.rank + 1) * 2].copy()
        spec = sf.exchange_strided_forward(buf, xp, ep)
        return spec.data.copy().real.reshape(2, 4), xp.counters.snapshot()

    res = sf.run_spmd(2, body, sf.CommMode.SERIAL)
    np.savez_compressed(os.path.join(HERE, "fig3_exchange.npz"),
                        p0=res[0][0], p1=res[1][0],
                        counters=np.array([r[1] for r in res]))
    print("wrote fig3_exchange.npz", res[0][0].tolist(), res[1][0].tolist())
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
