"""Full-size parity of the BASELINE configurations that bench.py times.

The oracle (oracle/slabfft_oracle.py, bit-identical to the reference path
dfft.py:148-215 on the golden fixtures) runs at FULL size on the GPU host's
cores; the GPU result of the same seeded input must match it within the
north_star tolerance (relative L2 <= 1e-12 float64, <= 1e-5 float32), per
rank in the STRIDED_INPLACE layout, and the forward -> inverse round trip must
recover the input to the same bound.  The reference is bitwise p-invariant
(SURVEY.md §8(c) step 1), so one p = 1 oracle spectrum G pins every p: rank
q's buffer is oracle.scatter_spectral(G, p)[q].

Configs (BASELINE.json): 512^3 float64 standard normal at p = 1, 2, 4 (p > 1
on the local fabric: p ranks on one GPU); 1024^3 float64 and float32 uniform
at p = 1 (the headline bench configuration; float32 gets the fp32-rounded
input) and float64 at p = 8 on the local fabric; the turbulence field (3 components, inverse
then forward) at 256^3 for p = 1, 2; and the per-rank shapes of 2048^3
over 8 ranks (config 4, which does not fit one GPU as a whole): 256 x 2048 x
2048 (rows of 2048, n1 = 2048 columns) and 2048 x 256 x 2048 (n0 = 2048
columns) at p = 1.  Comparisons run on the GPU (torch) to keep the 8.6 GB
buffers off the host's single-threaded numpy paths.
"""

import os

import numpy as np
import pytest
import torch

import oracle
import paper_1406_5597_b200 as tf

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
WORKERS = len(os.sched_getaffinity(0))
TOL = {"float64": 1e-12, "float32": 1e-5}


def rel_dev(got: torch.Tensor, ref) -> float:
    """relative L2 of got against ref (numpy or tensor), computed on got's device"""
    r = torch.as_tensor(ref).to(got.device).reshape(-1)
    g = got.reshape(-1).to(r.dtype)
    return float(torch.linalg.vector_norm(g - r) / torch.linalg.vector_norm(r))


@pytest.fixture(scope="module")
def n512():
    shape = (512, 512, 512)
    x = oracle.normal_field(shape, seed=3)
    g = oracle.forward_all(x, 1, workers=WORKERS)[0]  # p = 1 buffer == global spectrum, C order
    return x, g.reshape(512, 512, 257)


@pytest.mark.parametrize("p", [1, 2, 4])
def test_512_cubed_f64_vs_oracle(n512, p):
    x, G = n512
    shape = x.shape
    grid = tf.GlobalGrid(*shape)
    slabs = tf.scatter_real(x, grid, p)
    refs = oracle.scatter_spectral(G, p)

    def body(ep):
        fp = tf.plan(grid, ep, tf.Strategy.STRIDED)
        spec = tf.forward(fp, slabs[ep.rank])
        e_fwd = rel_dev(spec.data, refs[ep.rank])
        back = tf.inverse(fp, spec)
        e_rt = rel_dev(back.data, slabs[ep.rank].data)
        fp.close()
        return e_fwd, e_rt

    res = tf.run_spmd(p, body)
    for e_fwd, e_rt in res:
        assert e_fwd <= 1e-12 and e_rt <= 1e-12, res


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_1024_cubed_p1_vs_oracle(dtype):
    """The headline bench configuration, against the oracle at full size."""
    shape = (1024, 1024, 1024)
    x = oracle.uniform_field(shape, seed=11)
    if dtype == "float32":
        x = x.astype(np.float32).astype(np.float64)  # identical values on both sides
    ref = oracle.forward_all(x, 1, workers=WORKERS)[0]
    grid = tf.GlobalGrid(*shape)
    ep = tf.make_communicators(1)[0]
    fp = tf.plan(grid, ep, tf.Strategy.STRIDED, dtype=dtype)
    slab = tf.scatter_real(x, grid, 1, dtype=dtype)[0]
    del x
    spec = tf.forward(fp, slab)
    e_fwd = rel_dev(spec.data, ref)
    del ref
    back = tf.inverse(fp, spec)
    e_rt = rel_dev(back.data, slab.data)
    fp.close()
    assert e_fwd <= TOL[dtype], e_fwd
    assert e_rt <= TOL[dtype], e_rt


def test_1024_cubed_p8_local_fabric_vs_oracle():
    """The headline grid split over 8 ranks (local fabric: eight ranks on one
    B200), every rank's STRIDED_INPLACE buffer against the oracle's p = 1
    spectrum scattered to 8 ranks (the reference is bitwise p-invariant), and
    the round trip: the two-level column kernels, the band-redirecting stage
    1b and the exchange at the size north_star names for 8 GPUs."""
    shape, p = (1024, 1024, 1024), 8
    x = oracle.uniform_field(shape, seed=11)
    G = oracle.forward_all(x, 1, workers=WORKERS)[0].reshape(1024, 1024, 513)
    grid = tf.GlobalGrid(*shape)
    slabs = tf.scatter_real(x, grid, p)
    del x
    refs = oracle.scatter_spectral(G, p)
    del G

    def body(ep):
        fp = tf.plan(grid, ep, tf.Strategy.STRIDED)
        spec = tf.forward(fp, slabs[ep.rank])
        e_fwd = rel_dev(spec.data, refs[ep.rank])
        back = tf.inverse(fp, spec)
        e_rt = rel_dev(back.data, slabs[ep.rank].data)
        fp.close()
        return e_fwd, e_rt

    res = tf.run_spmd(p, body)
    for e_fwd, e_rt in res:
        assert e_fwd <= 1e-12 and e_rt <= 1e-12, res


@pytest.mark.parametrize("shape", [(256, 2048, 2048), (2048, 256, 2048)], ids=lambda v: "x".join(map(str, v)))
def test_2048_rank_shapes_p1_vs_oracle(shape):
    """BASELINE config 4 (2048^3 at p = 4, 8) per rank: the 8.6 GB real slab of
    one of 8 ranks.  2048-point rows and the 2 x 1024 tensor-memory column
    kernel (col_wpc2.cuh) on n1 (first shape) and on n0 (second shape), against
    the oracle at full size."""
    x = oracle.uniform_field(shape, seed=13)
    ref = oracle.forward_all(x, 1, workers=WORKERS)[0]
    grid = tf.GlobalGrid(*shape)
    ep = tf.make_communicators(1)[0]
    fp = tf.plan(grid, ep, tf.Strategy.STRIDED)
    slab = tf.scatter_real(x, grid, 1)[0]
    del x
    spec = tf.forward(fp, slab)
    e_fwd = rel_dev(spec.data, ref)
    del ref
    back = tf.inverse(fp, spec)
    e_rt = rel_dev(back.data, slab.data)
    fp.close()
    assert e_fwd <= 1e-12, e_fwd
    assert e_rt <= 1e-12, e_rt


@pytest.fixture(scope="module")
def turb256():
    """3 components of the turbulence field (BASELINE config 5 at 256^3, the
    shell scaled to 1 <= |k| <= 85) and the oracle's inverse of each."""
    shape = (256, 256, 256)
    amp = oracle.turbulence_amplitude(shape, 1.0, 340.0 * 256 / 1024)
    comps = []
    for c in range(3):
        noise = oracle.normal_field(shape, seed=100 + c)
        G = oracle.forward_all(noise, 1, workers=WORKERS)[0].reshape(256, 256, 129) * amp
        outs, _ = oracle.inverse_all(oracle.scatter_spectral(G, 1), shape, workers=WORKERS)
        comps.append((G, outs[0].reshape(shape)))
    return comps


@pytest.mark.parametrize("p", [1, 2])
def test_turbulence_256_vs_oracle(turb256, p):
    """inverse c2r of each component against the oracle's inverse, then
    forward r2c back to the spectrum (forward(inverse(G)) = G)."""
    shape = (256, 256, 256)
    grid = tf.GlobalGrid(*shape)
    specs = [tf.scatter_spectral(G, grid, p) for G, _ in turb256]
    reals = [tf.scatter_real(u, grid, p) for _, u in turb256]

    def body(ep):
        fp = tf.plan(grid, ep, tf.Strategy.STRIDED)
        errs = []
        for c in range(3):
            ref_spec = specs[c][ep.rank].data.clone()
            back = tf.inverse(fp, specs[c][ep.rank])
            errs.append(rel_dev(back.data, reals[c][ep.rank].data))
            spec = tf.forward(fp, back)
            errs.append(rel_dev(spec.data, ref_spec))
        fp.close()
        return errs

    for errs in tf.run_spmd(p, body):
        assert max(errs) <= 1e-12, errs
