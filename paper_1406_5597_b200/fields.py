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

from .dfft import DTYPES, FftPlan, forward, inverse
from .layout import RealSlab, SpectralSlab, SpectralTag

__all__ = ["radial_wavenumber", "turbulence_spectrum", "forward_batch", "inverse_batch"]


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


def turbulence_spectrum(fp: FftPlan, noise: RealSlab, kmin: float = 1.0, kmax: float = 340.0,
                        exponent: float = -5.0 / 3.0, out: torch.Tensor | None = None) -> SpectralSlab:
    """Collective.  ``noise`` is this rank's slab of a real white-noise field
    (any seeded generator); returns the shaped spectrum (forward of the noise
    times the radial amplitude), backed by ``out`` or plan memory."""
    spec = forward(fp, noise, out=out)
    kr = radial_wavenumber(fp)
    shell = (kr >= kmin) & (kr <= kmax)
    ksafe = torch.where(shell, kr, torch.ones_like(kr))
    amp = torch.where(shell, torch.sqrt(ksafe ** exponent / (4.0 * math.pi * ksafe ** 2)), torch.zeros_like(kr))
    rdt = DTYPES[fp.dtype][1]
    spec.data.mul_(amp.to(rdt))
    return SpectralSlab(fp.spectral_layout, SpectralTag.STRIDED_INPLACE, spec.data)


def inverse_batch(fp: FftPlan, specs: list[SpectralSlab], outs: list[torch.Tensor]) -> list[RealSlab]:
    """Batched inverse c2r of several components with one plan (consumes specs)."""
    return [inverse(fp, s, out=o) for s, o in zip(specs, outs)]


def forward_batch(fp: FftPlan, reals: list[RealSlab], outs: list[torch.Tensor]) -> list[SpectralSlab]:
    """Batched forward r2c of several components with one plan."""
    return [forward(fp, r, out=o) for r, o in zip(reals, outs)]
