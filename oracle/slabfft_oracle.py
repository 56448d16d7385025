"""CPU oracle for the transpose-free (STRIDED) slab 3D real FFT.

TEST INFRASTRUCTURE ONLY.  This module restates, in vectorised numpy, the
algorithm of the reference package ``slabfft`` 0.1.0 (``/root/reference/pkg``)
for the STRIDED strategy.  It is imported by ``tests/``, by
``__graft_entry__.smoke()`` (as the checker) and by ``bench.py``'s
cpu_baseline / ``--impl reference`` leg.  The product path
(``paper_1406_5597_b200``) never imports it.

Parity pin
----------
The reference's arithmetic is elementwise per row (kernels.py:134-140: "Row
results are bit-identical whether rows are transformed one at a time or
batched").  This restatement performs the same numpy ufunc sequence on
batches of rows, so its outputs are *bitwise identical* to the reference at
every grid and rank count.  ``tests/golden/make_golden.py`` imports the
reference from ``/root/reference/pkg/src`` and stores its outputs as golden
fixtures; ``tests/test_oracle.py`` checks this module against them bit for
bit.

The algorithm lives in numpy (a third-party dependency of the reference,
pinned ``numpy>=1.24`` in pkg/pyproject.toml:10; 2.3.5 here): radix-2 DIT
with a bit-reversal gather and complex-multiply / add / subtract ufuncs.
"""

from __future__ import annotations

import functools
from concurrent.futures import ThreadPoolExecutor

import numpy as np

__all__ = [
    "OracleConsistencyError",
    "twiddles",
    "bitrev_perm",
    "c2c_rows",
    "r2c_rows",
    "c2r_rows",
    "stage1_forward",
    "stage1_inverse",
    "strided_column_offsets",
    "exchange_strided",
    "stage3",
    "forward_all",
    "inverse_all",
    "gather_spectral",
    "scatter_spectral",
    "spectral_offset",
    "dft3d_r2c_naive",
    "dft1d_naive",
    "uniform_field",
    "normal_field",
    "stage1_band_staging",
    "turbulence_amplitude",
]

C2R_RESIDUE_TOL = 1e-9  # kernels.py:38


class OracleConsistencyError(ValueError):
    """Mirror of slabfft ConsistencyError (errors.py:32-33)."""


# ---------------------------------------------------------------------------
# 1D kernels (kernels.py)
# ---------------------------------------------------------------------------

@functools.lru_cache(maxsize=None)
def twiddles(n: int) -> np.ndarray:
    """exp(-2*pi*i*k/n) for k < n/2, exactly as kernels.py:76-81 builds it."""
    return np.exp(-2j * np.pi * np.arange(n // 2) / n)


@functools.lru_cache(maxsize=None)
def bitrev_perm(n: int) -> np.ndarray:
    """Bit-reversal permutation of [0, n) (kernels.py:53-61)."""
    bits = n.bit_length() - 1
    idx = np.arange(n)
    out = np.zeros(n, dtype=np.intp)
    for b in range(bits):
        out |= ((idx >> b) & 1) << (bits - 1 - b)
    return out


def c2c_rows(a: np.ndarray, inverse: bool) -> None:
    """In-place unnormalised radix-2 DIT over the last axis of a 2D C-order
    complex128 array (kernels.py:134-161).  Forward uses exp(-2*pi*i...)."""
    rows, n = a.shape
    if n < 2:
        return
    a[:] = a[:, bitrev_perm(n)]
    tab = twiddles(n)
    half = 1
    while half < n:
        span = 2 * half
        w = tab[:: n // span]
        if inverse:
            w = w.conj()
        grp = a.reshape(rows, n // span, span)
        lo = grp[:, :, :half]
        hi = grp[:, :, half:]
        t = hi * w
        np.subtract(lo, t, out=hi)
        np.add(lo, t, out=lo)
        half = span


def r2c_rows(rows: np.ndarray) -> np.ndarray:
    """Half-spectrum transform of each real row (kernels.py:203-209)."""
    n = rows.shape[1]
    work = rows.astype(np.complex128)
    c2c_rows(work, inverse=False)
    return np.ascontiguousarray(work[:, : n // 2 + 1])


def c2r_rows(half: np.ndarray, n: int) -> tuple[np.ndarray, float]:
    """Unnormalised inverse of r2c_rows for one plane's rows, with the
    reference's Hermitian consistency checks (kernels.py:212-239)."""
    n2c = n // 2 + 1
    scale = float(np.max(np.abs(half))) if half.size else 0.0
    tol = C2R_RESIDUE_TOL * n * scale
    edge = max(np.max(np.abs(half[:, 0].imag)), np.max(np.abs(half[:, n // 2].imag)))
    if edge > tol:
        raise OracleConsistencyError(f"edge bins not real: {edge:.3e} > {tol:.3e}")
    full = np.empty((half.shape[0], n), dtype=np.complex128)
    full[:, :n2c] = half
    full[:, n2c:] = half[:, 1 : n // 2][:, ::-1].conj()
    c2c_rows(full, inverse=True)
    residue = float(np.max(np.abs(full.imag)))
    if residue > tol:
        raise OracleConsistencyError(f"imag residue {residue:.3e} > {tol:.3e}")
    return np.ascontiguousarray(full.real), residue


# ---------------------------------------------------------------------------
# stage 1 / 1' : per-plane 2D transforms (kernels.py:262-303, dfft.py:161-163, 205-209)
# ---------------------------------------------------------------------------

def _chunks(count: int, workers: int, max_step: int | None = None):
    """Spans of [0, count) for `workers` threads; `max_step` bounds a span so
    the per-span temporaries stay small at full size (1024^3).  Batching rows
    differently does not change a bit of the result (kernels.py:134-140)."""
    workers = max(1, min(workers, count))
    step = -(-count // workers)
    if max_step:
        step = max(1, min(step, max_step))
    return [(a, min(a + step, count)) for a in range(0, count, step)]


def _run(fn, spans, workers):
    if workers <= 1 or len(spans) <= 1:
        return [fn(a, b) for a, b in spans]
    with ThreadPoolExecutor(max_workers=workers) as ex:
        return list(ex.map(lambda s: fn(*s), spans))


def stage1_forward(slab: np.ndarray, workers: int = 1) -> np.ndarray:
    """(n0p, n1, n2) real -> (n0p, n1, n2c) complex: r2c along n2 of every
    row, then forward c2c along n1 of every retained column, per plane."""
    n0p, n1, n2 = slab.shape
    n2c = n2 // 2 + 1
    out = np.empty((n0p, n1, n2c), dtype=np.complex128)

    def work(a, b):
        half = r2c_rows(slab[a:b].reshape(-1, n2)).reshape(b - a, n1, n2c)
        cols = np.ascontiguousarray(half.transpose(0, 2, 1)).reshape(-1, n1)
        c2c_rows(cols, inverse=False)
        out[a:b] = cols.reshape(b - a, n2c, n1).transpose(0, 2, 1)

    _run(work, _chunks(n0p, workers, max(1, (1 << 22) // (n1 * n2))), workers)
    return out


def stage1_inverse(buf: np.ndarray, n2: int, workers: int = 1) -> tuple[np.ndarray, float]:
    """(n0p, n1, n2c) complex -> (n0p, n1, n2) real, unnormalised, per-plane
    consistency check; returns (real, max imag residue)."""
    n0p, n1, n2c = buf.shape
    out = np.empty((n0p, n1, n2), dtype=np.float64)

    def work(a, b):
        res = 0.0
        for i in range(a, b):
            cols = np.ascontiguousarray(buf[i].T)
            c2c_rows(cols, inverse=True)
            half = np.ascontiguousarray(cols.T)
            real, r = c2r_rows(half, n2)
            out[i] = real
            res = max(res, r)
        return res

    res = _run(work, _chunks(n0p, workers, max(1, (1 << 22) // (n1 * n2))), workers)
    return out, max(res) if res else 0.0


# ---------------------------------------------------------------------------
# STRIDED_INPLACE layout, exchange, stage 3 (layout.py:189-219, exchange.py:106-121, 263-290)
# ---------------------------------------------------------------------------

def spectral_offset(n0: int, n1: int, n2: int, p: int, j: int, r: int, k: int) -> int:
    """Buffer offset of logical (j, r, k) in a STRIDED_INPLACE slab (layout.py:197-198)."""
    n0p, n1p, n2c = n0 // p, n1 // p, n2 // 2 + 1
    return (r % n0p) * (n1 * n2c) + (r // n0p) * (n1p * n2c) + j * n2c + k


def strided_column_offsets(n0: int, n1: int, n2: int, p: int) -> np.ndarray:
    """(ncols, n0) offsets; row c is the TwoLevelStride of column c = j*n2c+k
    (layout.py:201-219 with kernels.py:112-124)."""
    n0p, n1p, n2c = n0 // p, n1 // p, n2 // 2 + 1
    r = np.arange(n0)
    col = (r % n0p) * (n1 * n2c) + (r // n0p) * (n1p * n2c)
    c = np.arange(n1p * n2c)
    return c[:, None] + col[None, :]


def exchange_strided(bufs: list[np.ndarray]) -> None:
    """In-place band swap among p ranks' (n0p, n1, n2c) buffers: rank s's
    band q trades places with rank q's band s (exchange.py:114-121, 275, 289).
    The same call is the forward and the inverse exchange."""
    p = len(bufs)
    n1p = bufs[0].shape[1] // p
    for s in range(p):
        for q in range(s + 1, p):
            a = bufs[s][:, q * n1p : (q + 1) * n1p]
            b = bufs[q][:, s * n1p : (s + 1) * n1p]
            tmp = a.copy()
            a[...] = b
            b[...] = tmp


def stage3(flat: np.ndarray, n0: int, n1: int, n2: int, p: int, inverse: bool,
           workers: int = 1) -> None:
    """Length-n0 c2c over every owned column, gathered by its two-level
    stride, transformed and scattered back (kernels.py:176-200, dfft.py:170-171, 196-197)."""
    n0p, n1p, n2c = n0 // p, n1 // p, n2 // 2 + 1
    r = np.arange(n0, dtype=np.int64)
    col = (r % n0p) * (n1 * n2c) + (r // n0p) * (n1p * n2c)  # TwoLevelStride of column 0

    def work(a, b):
        # rows a..b of strided_column_offsets, built per span (the full table is
        # ncols x n0 int64: 4.3 GB at 1024^3)
        offs = np.arange(a, b, dtype=np.int64)[:, None] + col[None, :]
        cols = flat[offs]
        c2c_rows(cols, inverse)
        flat[offs] = cols

    _run(work, _chunks(n1p * n2c, workers, max(1, (1 << 22) // n0)), workers)


def forward_all(field: np.ndarray, p: int, workers: int = 1) -> list[np.ndarray]:
    """Run dfft.forward (dfft.py:148-176, STRIDED) on all p ranks; returns
    each rank's flat complex128 STRIDED_INPLACE buffer."""
    n0, n1, n2 = field.shape
    n0p = n0 // p
    bufs = [stage1_forward(np.ascontiguousarray(field[s * n0p : (s + 1) * n0p]), workers)
            for s in range(p)]
    exchange_strided(bufs)
    flats = [b.reshape(-1) for b in bufs]
    for f in flats:
        stage3(f, n0, n1, n2, p, inverse=False, workers=workers)
    return flats


def inverse_all(flats: list[np.ndarray], shape: tuple[int, int, int],
                workers: int = 1) -> tuple[list[np.ndarray], float]:
    """Run dfft.inverse (dfft.py:179-215, STRIDED) on all ranks.  Consumes
    ``flats`` in place; returns per-rank (n0p, n1, n2) real slabs and the max
    imaginary residue."""
    n0, n1, n2 = shape
    p = len(flats)
    n0p, n2c = n0 // p, n2 // 2 + 1
    for f in flats:
        stage3(f, n0, n1, n2, p, inverse=True, workers=workers)
    bufs = [f.reshape(n0p, n1, n2c) for f in flats]
    exchange_strided(bufs)
    outs, res = [], 0.0
    for b in bufs:
        real, r = stage1_inverse(b, n2, workers)
        real *= 1.0 / (n0 * n1 * n2)
        outs.append(real)
        res = max(res, r)
    return outs, res


def gather_spectral(flats: list[np.ndarray], shape: tuple[int, int, int]) -> np.ndarray:
    """Global (n0, n1, n2c) spectrum from p STRIDED_INPLACE buffers (dfft.py:218-238)."""
    n0, n1, n2 = shape
    p = len(flats)
    n0p, n1p, n2c = n0 // p, n1 // p, n2 // 2 + 1
    out = np.empty((n0, n1, n2c), dtype=flats[0].dtype)
    for q, f in enumerate(flats):
        v = f.reshape(n0p, p, n1p, n2c)  # [i][s][j][k] = G[s*n0p+i, q*n1p+j, k]
        out[:, q * n1p : (q + 1) * n1p, :] = v.transpose(1, 0, 2, 3).reshape(n0, n1p, n2c)
    return out


def scatter_spectral(glob: np.ndarray, p: int) -> list[np.ndarray]:
    """Inverse of gather_spectral: per-rank STRIDED_INPLACE flat buffers."""
    n0, n1, n2c = glob.shape
    n0p, n1p = n0 // p, n1 // p
    outs = []
    for q in range(p):
        band = glob[:, q * n1p : (q + 1) * n1p, :].reshape(p, n0p, n1p, n2c)
        outs.append(band.transpose(1, 0, 2, 3).copy().reshape(-1))  # always a copy: inverse_all consumes it
    return outs


def stage1_band_staging(stage1_out: np.ndarray, p: int, rank: int):
    """Where the GPU stage-1 epilogue puts each band before the exchange:
    the self band stays in place, band q != rank goes to staging[q][i][j][k]
    (contiguous per (q, i) chunk).  Returns (inplace_buffer, staging)."""
    n0p, n1, n2c = stage1_out.shape
    n1p = n1 // p
    staging = np.zeros((p, n0p, n1p, n2c), dtype=stage1_out.dtype)
    inplace = np.zeros_like(stage1_out)
    inplace[:, rank * n1p : (rank + 1) * n1p] = stage1_out[:, rank * n1p : (rank + 1) * n1p]
    for q in range(p):
        if q != rank:
            staging[q] = stage1_out[:, q * n1p : (q + 1) * n1p]
    return inplace, staging


# ---------------------------------------------------------------------------
# brute-force oracle (oracle.py:17-45) and seeded inputs (cli.py:78-80)
# ---------------------------------------------------------------------------

def _basis(n: int, sign: float) -> np.ndarray:
    k = np.arange(n)
    return np.exp(sign * 2j * np.pi * np.outer(k, k) / n)


def dft1d_naive(x: np.ndarray, inverse: bool = False) -> np.ndarray:
    x = np.asarray(x, dtype=np.complex128)
    return _basis(x.shape[0], 1.0 if inverse else -1.0) @ x


def dft3d_r2c_naive(f: np.ndarray) -> np.ndarray:
    """Direct triple sum, truncated to n2/2+1 bins (oracle.py:30-45)."""
    f = np.asarray(f, dtype=np.float64)
    n0, n1, n2 = f.shape
    e2 = np.exp(-2j * np.pi * np.outer(np.arange(n2 // 2 + 1), np.arange(n2)) / n2)
    return np.einsum("ai,bj,ck,ijk->abc", _basis(n0, -1.0), _basis(n1, -1.0), e2,
                     f.astype(np.complex128), optimize=False)


def uniform_field(shape, seed: int) -> np.ndarray:
    """iid uniform[-1, 1) from numpy default_rng(seed), C order."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=shape)


def normal_field(shape, seed: int) -> np.ndarray:
    """iid standard normal from default_rng(seed) (cli.py:78-80)."""
    return np.random.default_rng(seed).standard_normal(shape)


def turbulence_amplitude(shape, kmin=1.0, kmax=340.0, exponent=-5.0 / 3.0) -> np.ndarray:
    """Global (n0, n1, n2c) radial amplitude sqrt(E(|k|) / (4 pi |k|^2)) on the
    shell kmin <= |k| <= kmax, signed frequencies on axes 0 and 1 (the
    turbulence configuration of BASELINE.json)."""
    n0, n1, n2 = shape
    f0 = np.fft.fftfreq(n0, 1.0 / n0)
    f1 = np.fft.fftfreq(n1, 1.0 / n1)
    f2 = np.arange(n2 // 2 + 1, dtype=np.float64)
    k = np.sqrt(f0[:, None, None] ** 2 + f1[None, :, None] ** 2 + f2[None, None, :] ** 2)
    shell = (k >= kmin) & (k <= kmax)
    ks = np.where(shell, k, 1.0)
    return np.where(shell, np.sqrt(ks ** exponent / (4.0 * np.pi * ks ** 2)), 0.0)
