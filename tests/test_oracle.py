"""The CPU oracle, pinned against the reference.

* bit-exact against the golden fixtures produced by the unmodified reference
  (tests/golden/make_golden.py);
* the reference's own known-answer tests (pkg/tests/test_kernels.py) and the
  SPEC/paper Fig. 3 exchange vector, restated here.
"""

import glob
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CASES = sorted(glob.glob(os.path.join(GOLDEN, "ref_*.npz")))


def _field(d):
    gen = oracle.uniform_field if str(d["dist"]) == "uniform" else oracle.normal_field
    return gen(tuple(int(v) for v in d["shape"]), int(d["seed"]))


@pytest.mark.parametrize("path", CASES, ids=os.path.basename)
def test_oracle_bitwise_equals_reference(path):
    d = np.load(path)
    x = _field(d)
    p = int(d["p"])
    fwd = oracle.forward_all(x, p)
    for q in range(p):
        assert np.array_equal(fwd[q].view(np.float64), d["fwd"][q].view(np.float64))
    outs, res = oracle.inverse_all([f.copy() for f in fwd], x.shape)
    for q in range(p):
        assert np.array_equal(outs[q].reshape(-1), d["inv"][q])
    assert res == float(d["residue"])


def test_golden_fixture_count():
    assert len(CASES) >= 10


# --- reference known answers (pkg/tests/test_kernels.py) -------------------

def c2c(values, inverse=False):
    a = np.asarray(values, dtype=np.complex128).reshape(1, -1).copy()
    oracle.c2c_rows(a, inverse)
    return a[0]


def test_twiddles():
    np.testing.assert_allclose(oracle.twiddles(4), [1.0, -1.0j], atol=1e-15)
    assert abs(oracle.twiddles(8)[1] - np.sqrt(2) / 2 * (1 - 1j)) < 1e-15
    assert oracle.twiddles(1).size == 0


def test_c2c_known_answers():
    np.testing.assert_allclose(c2c([1, 0, 0, 0]), [1, 1, 1, 1], atol=0)
    np.testing.assert_allclose(c2c([1, 1, 1, 1]), [4, 0, 0, 0], atol=1e-15)
    np.testing.assert_allclose(c2c([0, 1, 0, 0]), [1, -1j, -1, 1j], atol=1e-15)


@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_c2c_matches_naive(n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    assert np.max(np.abs(c2c(x) - oracle.dft1d_naive(x))) <= 1e-12 * n


@pytest.mark.parametrize("n", [2, 8, 64])
def test_inverse_unnormalised_and_parseval(n):
    rng = np.random.default_rng(n + 1)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    X = c2c(x)
    np.testing.assert_allclose(c2c(X, inverse=True), n * x, atol=1e-12 * n)
    assert abs(np.sum(np.abs(X) ** 2) - n * np.sum(np.abs(x) ** 2)) <= 1e-10 * n * np.sum(np.abs(x) ** 2)


def test_real_transforms_known_answers():
    np.testing.assert_allclose(oracle.r2c_rows(np.array([[1.0, 1, 1, 1]]))[0], [4, 0, 0], atol=1e-15)
    np.testing.assert_allclose(oracle.r2c_rows(np.array([[1.0, 0, 0, 0]]))[0], [1, 1, 1], atol=1e-15)
    np.testing.assert_allclose(oracle.r2c_rows(np.array([[0.0, 1, 0, 1]]))[0], [2, 0, -2], atol=1e-15)
    real, _ = oracle.c2r_rows(np.array([[4.0 + 0j, 0, 0]]), 4)
    np.testing.assert_allclose(real[0], [4, 4, 4, 4], atol=1e-15)
    real, _ = oracle.c2r_rows(np.array([[1.0 + 0j, 1, 1]]), 4)
    np.testing.assert_allclose(real[0], [4, 0, 0, 0], atol=1e-15)


def test_c2r_rejects_corrupted_spectrum():
    with pytest.raises(oracle.OracleConsistencyError):
        oracle.c2r_rows(np.array([[1.0 + 1j, 0, 0]]), 4)


def test_3d_against_brute_force():
    x = oracle.normal_field((4, 8, 4), 3)
    for p in (1, 2, 4):
        got = oracle.gather_spectral(oracle.forward_all(x, p), x.shape)
        assert np.max(np.abs(got - oracle.dft3d_r2c_naive(x))) <= 1e-10


def test_constant_and_delta_fields():
    """SPEC.md constant -> DC and delta -> all-ones examples."""
    x = np.ones((4, 4, 4))
    g = oracle.gather_spectral(oracle.forward_all(x, 2), x.shape)
    want = np.zeros_like(g)
    want[0, 0, 0] = 64
    np.testing.assert_allclose(g, want, atol=1e-12)
    d = np.zeros((4, 4, 4))
    d[0, 0, 0] = 1
    g = oracle.gather_spectral(oracle.forward_all(d, 2), d.shape)
    np.testing.assert_allclose(g, np.ones_like(g), atol=1e-15)


def test_fig3_exchange_vector():
    """Paper Fig. 3 / SPEC.md:548: 4x4 (n2c=1), p=2, STRIDED in-place exchange."""
    fig = np.load(os.path.join(GOLDEN, "fig3_exchange.npz"))
    bufs = [np.arange(1, 9, dtype=np.complex128).reshape(2, 4, 1),
            np.arange(9, 17, dtype=np.complex128).reshape(2, 4, 1)]
    oracle.exchange_strided(bufs)
    np.testing.assert_array_equal(bufs[0].real.reshape(2, 4), [[1, 2, 9, 10], [5, 6, 13, 14]])
    np.testing.assert_array_equal(bufs[0].real.reshape(2, 4), fig["p0"])
    np.testing.assert_array_equal(bufs[1].real.reshape(2, 4), fig["p1"])
    # STRIDED: nothing packed or unpacked, each rank puts 4 complex128 on the wire
    assert fig["counters"].tolist() == [[0, 64, 0], [0, 64, 0]]


def test_scatter_gather_spectral_roundtrip():
    rng = np.random.default_rng(0)
    g = rng.standard_normal((8, 8, 5)) + 1j * rng.standard_normal((8, 8, 5))
    for p in (1, 2, 4, 8):
        assert np.array_equal(oracle.gather_spectral(oracle.scatter_spectral(g, p), (8, 8, 8)), g)


def test_strided_offsets_match_spectral_offset():
    n0, n1, n2, p = 8, 4, 6, 2
    offs = oracle.strided_column_offsets(n0, n1, n2, p)
    n2c = n2 // 2 + 1
    for c in range(offs.shape[0]):
        j, k = divmod(c, n2c)
        assert list(offs[c]) == [oracle.spectral_offset(n0, n1, n2, p, j, r, k) for r in range(n0)]


# --- further restatements of pkg/tests/test_kernels.py --------------------

def test_c2c_linearity():
    """TestC2C linearity (test_kernels.py:53-113)."""
    rng = np.random.default_rng(5)
    x = rng.standard_normal(16) + 1j * rng.standard_normal(16)
    y = rng.standard_normal(16) + 1j * rng.standard_normal(16)
    a, b = 2.5 - 1j, -0.75 + 0.5j
    np.testing.assert_allclose(c2c(a * x + b * y), a * c2c(x) + b * c2c(y), atol=1e-12)


def test_r2c_edge_bins_real_and_hermitian_embedding():
    """TestRealTransforms (test_kernels.py:179-234): the DC and Nyquist bins of
    a real row are real, and r2c equals the first n/2+1 bins of the full c2c."""
    rng = np.random.default_rng(9)
    x = rng.standard_normal((3, 16))
    half = oracle.r2c_rows(x)
    assert half.shape == (3, 9)
    assert np.all(half[:, 0].imag == 0) and np.max(np.abs(half[:, 8].imag)) <= 1e-14
    full = x.astype(np.complex128)
    oracle.c2c_rows(full, False)
    np.testing.assert_allclose(half, full[:, :9], atol=1e-13)


def test_real_round_trip_is_unnormalised():
    """c2r(r2c(x)) = n x (test_kernels.py: unnormalised round trip, 8 x at n = 8)."""
    rng = np.random.default_rng(11)
    x = rng.standard_normal((2, 8))
    back, _ = oracle.c2r_rows(oracle.r2c_rows(x), 8)
    np.testing.assert_allclose(back, 8 * x, atol=1e-12)


def test_plane_transform_vs_naive_2d():
    """TestPlaneTransforms (test_kernels.py:237-268): a 4 x 4 plane r2c
    against a naive 2D DFT, and the plane round trip x n1 n2."""
    rng = np.random.default_rng(13)
    plane = rng.standard_normal((1, 4, 4))
    got = oracle.stage1_forward(plane)
    want = np.stack([oracle.dft1d_naive(col) for col in
                     np.stack([oracle.dft1d_naive(r)[:3] for r in plane[0]]).T]).T
    assert np.max(np.abs(got.reshape(4, 3) - want)) <= 1e-12
    back, _ = oracle.stage1_inverse(got.copy(), 4)
    np.testing.assert_allclose(back.reshape(4, 4), 16 * plane[0], atol=1e-12)


def test_stage3_equals_gather_fft_scatter():
    """TestC2CStrided (test_kernels.py:141-158): the strided column FFT is
    bitwise the gather -> FFT -> scatter of the same column."""
    n0, n1, n2, p = 8, 4, 4, 2
    rng = np.random.default_rng(17)
    n2c = n2 // 2 + 1
    flat = rng.standard_normal((n1 // p) * n0 * n2c) + 1j * rng.standard_normal((n1 // p) * n0 * n2c)
    offs = oracle.strided_column_offsets(n0, n1, n2, p)
    want = flat.copy()
    cols = want[offs].copy()
    oracle.c2c_rows(cols, False)
    want[offs] = cols
    got = flat.copy()
    oracle.stage3(got, n0, n1, n2, p, inverse=False)
    assert np.array_equal(got.view(np.float64), want.view(np.float64))
