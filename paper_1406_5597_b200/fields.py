"""Synthetic fields for the BASELINE configurations, built on the device.

``turbulence_spectrum`` makes BASELINE.json config 5: a velocity component
defined in Fourier space with random phases and energy spectrum
E(k) ~ k^(-5/3) on kmin <= |k| <= kmax (zero elsewhere).  The reference has no
spectrum generator and its c2r rejects non-Hermitian input (kernels.py:225-238),
so the phases come from the transform of real white noise (exactly Hermitian
on the k2 = 0 and k2 = n2/2 planes) and are scaled by a real radial amplitude
sqrt(E(|k|) / (4 pi |k|^2)).  Signed frequencies are
used on axes 0 and 1.  The spectral slab is in the STRIDED_INPLACE layout of
the plan's rank.
"""

from __future__ import annotations

import math

import torch

from .dfft import DTYPES, FftPlan, forward, forward_many, inverse, inverse_many
from .errors import ContractError
from .layout import RealSlab, SpectralSlab, SpectralTag

__all__ = ["radial_wavenumber", "turbulence_spectrum", "turbulence_spectra", "forward_batch", "inverse_batch"]


def radial_wavenumber(fp: FftPlan, dtype=torch.float64) -> torch.Tensor:
    """|k| of every element of this rank's STRIDED_INPLACE spectral buffer,
    as a flat tensor in buffer order: element [i][s][j][k2] holds global bin
    (r = s*n0p + i, c = rank*n1p + j, k2)."""
    g = fp.grid
    p, rank = fp.p, fp.rank
    n0p, n1p, n2c = g.n0 // p, g.n1 // p, g.n2c
    dev = fp.device
    i = torch.arange(n0p, device=dev)
    s = torch.arange(p, device=dev)
    r = (s[None, :] * n0p + i[:, None])  # (n0p, p)
    f0 = torch.where(r < g.n0 // 2, r, r - g.n0).to(dtype)
    c = rank * n1p + torch.arange(n1p, device=dev)
    f1 = torch.where(c < g.n1 // 2, c, c - g.n1).to(dtype)
    f2 = torch.arange(n2c, device=dev, dtype=dtype)
    k2 = (f0[:, :, None, None] ** 2 + f1[None, None, :, None] ** 2 + f2[None, None, None, :] ** 2)
    return torch.sqrt(k2).reshape(-1)


def _amplitude(fp: FftPlan, kmin: float, kmax: float, exponent: float) -> torch.Tensor:
    kr = radial_wavenumber(fp)
    shell = (kr >= kmin) & (kr <= kmax)
    ksafe = torch.where(shell, kr, torch.ones_like(kr))
    amp = torch.where(shell, torch.sqrt(ksafe ** exponent / (4.0 * math.pi * ksafe ** 2)), torch.zeros_like(kr))
    return amp.to(DTYPES[fp.dtype][1])


def turbulence_spectrum(fp: FftPlan, noise: RealSlab, kmin: float = 1.0, kmax: float = 340.0,
                        exponent: float = -5.0 / 3.0, out: torch.Tensor | None = None) -> SpectralSlab:
    """Collective.  ``noise`` is this rank's slab of a real white-noise field
    (any seeded generator); returns the shaped spectrum (forward of the noise
    times the radial amplitude), backed by ``out`` or plan memory."""
    spec = forward(fp, noise, out=out)
    spec.data.mul_(_amplitude(fp, kmin, kmax, exponent))
    return SpectralSlab(fp.spectral_layout, SpectralTag.STRIDED_INPLACE, spec.data)


def turbulence_spectra(fp: FftPlan, noise: torch.Tensor, kmin: float = 1.0, kmax: float = 340.0,
                       exponent: float = -5.0 / 3.0, out: torch.Tensor | None = None) -> torch.Tensor:
    """Batched plan: ``noise`` holds ``fp.batch`` white-noise real slabs back
    to back; returns the ``fp.batch`` shaped spectra back to back."""
    spec = forward_many(fp, noise, out=out)
    spec.view(fp.batch, -1).mul_(_amplitude(fp, kmin, kmax, exponent))
    return spec


def _contiguous_run(ts: list[torch.Tensor]) -> torch.Tensor | None:
    """The one tensor the list is a back-to-back run of, or None."""
    base, n = ts[0], ts[0].numel()
    step = n * base.element_size()
    for i, t in enumerate(ts):
        if t.numel() != n or not t.is_contiguous() or t.data_ptr() != base.data_ptr() + i * step:
            return None
    return torch.as_strided(base, (len(ts) * n,), (1,))


def inverse_batch(fp: FftPlan, specs: list, outs: list[torch.Tensor] | None = None) -> list[RealSlab]:
    """Inverse c2r of several fields (consumes specs).  A batched plan
    (``fp.batch == len(specs)``) runs them in one library call -- one launch
    per stage at p = 1, exchange/compute overlap at p > 1 -- when the spectra
    are back-to-back views of one buffer (else they are gathered first)."""
    data = [s.data if isinstance(s, SpectralSlab) else s for s in specs]
    if fp.batch == 1:
        outs = outs or [None] * len(data)
        return [inverse(fp, SpectralSlab(fp.spectral_layout, SpectralTag.STRIDED_INPLACE, d), out=o)
                for d, o in zip(data, outs)]
    if len(data) != fp.batch:
        raise ContractError(f"plan has batch={fp.batch}, got {len(data)} fields")
    run = _contiguous_run(data)
    if run is None:
        run = torch.cat([d.reshape(-1) for d in data])
    dst = None if outs is None else _contiguous_run(outs)
    if outs is not None and dst is None:
        raise ContractError("outputs must be back-to-back views of one buffer")
    res = inverse_many(fp, run, out=dst).view(fp.batch, -1)
    return [RealSlab(fp.real_layout, res[c]) for c in range(fp.batch)]


def forward_batch(fp: FftPlan, reals: list, outs: list[torch.Tensor] | None = None) -> list[SpectralSlab]:
    """Forward r2c of several fields (see inverse_batch)."""
    data = [r.data if isinstance(r, RealSlab) else r for r in reals]
    if fp.batch == 1:
        outs = outs or [None] * len(data)
        return [forward(fp, RealSlab(fp.real_layout, d), out=o) for d, o in zip(data, outs)]
    if len(data) != fp.batch:
        raise ContractError(f"plan has batch={fp.batch}, got {len(data)} fields")
    run = _contiguous_run(data)
    if run is None:
        run = torch.cat([d.reshape(-1) for d in data])
    dst = None if outs is None else _contiguous_run(outs)
    if outs is not None and dst is None:
        raise ContractError("outputs must be back-to-back views of one buffer")
    res = forward_many(fp, run, out=dst).view(fp.batch, -1)
    return [SpectralSlab(fp.spectral_layout, SpectralTag.STRIDED_INPLACE, res[c]) for c in range(fp.batch)]
