"""Host-side mirror of slabfft.layout / dfft helpers (no GPU)."""

import numpy as np
import pytest
import torch

import oracle
import paper_1406_5597_b200 as tf


def test_grid_and_validate():
    g = tf.GlobalGrid(8, 4, 8)
    assert g.n2c == 5 and g.points == 256
    with pytest.raises(tf.ConfigurationError):
        tf.GlobalGrid(6, 4, 4)
    with pytest.raises(tf.ConfigurationError):
        tf.validate(tf.GlobalGrid(8, 8, 1), 1)
    with pytest.raises(tf.ConfigurationError):
        tf.validate(tf.GlobalGrid(8, 4, 4), 8)
    tf.validate(tf.GlobalGrid(8, 8, 8), 8)


def test_owned_range_and_shapes():
    g = tf.GlobalGrid(16, 8, 4)
    lay = tf.SlabLayout(g, 4, 2, tf.DistAxis.REAL_AXIS0)
    assert tf.owned_range(lay) == (8, 4) and lay.local_shape() == (4, 8, 4)
    lay = tf.SlabLayout(g, 4, 2, tf.DistAxis.SPECTRAL_AXIS1)
    assert tf.owned_range(lay) == (4, 2) and lay.local_shape() == (2, 16, 3)


def test_spectral_offset_and_column_descriptor_match_oracle():
    g = tf.GlobalGrid(8, 4, 8)
    p, rank = 2, 1
    lay = tf.SlabLayout(g, p, rank, tf.DistAxis.SPECTRAL_AXIS1)
    slab = tf.SpectralSlab(lay, tf.SpectralTag.STRIDED_INPLACE,
                           torch.zeros(lay.n1p * g.n0 * g.n2c, dtype=torch.complex128))
    for j in range(lay.n1p):
        for k in range(g.n2c):
            d = tf.column_stride_descriptor(slab, j, k)
            assert d.offsets() == [tf.spectral_offset(slab, j, r, k) for r in range(g.n0)]
            assert d.offsets() == [oracle.spectral_offset(g.n0, g.n1, g.n2, p, j, r, k) for r in range(g.n0)]


def test_as_logical_matches_gather():
    rng = np.random.default_rng(1)
    glob = rng.standard_normal((8, 8, 5)) + 1j * rng.standard_normal((8, 8, 5))
    slabs = tf.scatter_spectral(glob, tf.GlobalGrid(8, 8, 8), 4, device="cpu")
    assert np.array_equal(tf.gather_spectral(slabs), glob)
    flats = oracle.scatter_spectral(glob, 4)
    for s, f in zip(slabs, flats):
        assert np.array_equal(s.data.numpy(), f)


def test_real_scatter_gather():
    x = np.random.default_rng(2).standard_normal((8, 4, 4))
    slabs = tf.scatter_real(x, tf.GlobalGrid(8, 4, 4), 4, device="cpu")
    assert np.array_equal(tf.gather_real(slabs), x)
    with pytest.raises(tf.ContractError):
        tf.RealSlab(slabs[0].layout, torch.zeros(3, dtype=torch.float64))
    with pytest.raises(tf.ContractError):
        tf.RealSlab(slabs[0].layout, torch.zeros(32, dtype=torch.int32))


def test_plan_rejects_unknown_comm_pattern_without_gpu():
    with pytest.raises(tf.ConfigurationError):
        tf.plan(tf.GlobalGrid(8, 8, 8), type("E", (), {"p": 1, "rank": 0})(), tf.Strategy.STRIDED,
                "collective")
