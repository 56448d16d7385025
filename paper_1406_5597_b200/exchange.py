"""Exchange strategies and the STRIDED exchange geometry (mirror of
slabfft.exchange, reference pkg/src/slabfft/exchange.py:48-121).

On the GPU the exchange itself runs inside libtffft (NCCL grouped
send/recv, or the local fabric's device pull); this module exposes the
strategy enum and the per-rank chunk schedule the library executes, so the
geometry can be checked without a GPU (tests/test_exchange_gloo.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from enum import Enum

from . import _lib

__all__ = ["Strategy", "ExchangeOp", "exchange_schedule"]


class Strategy(Enum):
    TRANSPOSE = "transpose"
    STRIDED = "strided"


@dataclass(frozen=True)
class ExchangeOp:
    """One peer of the STRIDED exchange: ``count`` complex elements (the
    n0/p chunks of (n1/p)*n2c of the reference's LayoutDescriptor(count=n0/p,
    block_length=(n1/p)*n2c, stride=n1*n2c, base=q*(n1/p)*n2c),
    exchange.py:114-119) go from staging[send_offset] to the peer, and the
    peer's band for this rank arrives at landing[recv_offset].  The FFT stage
    after the exchange reads the landing band through the STRIDED_INPLACE
    addressing, so no rearrangement pass follows."""

    peer: int
    send_offset: int
    recv_offset: int
    count: int


def exchange_schedule(n0: int, n1: int, n2: int, p: int, rank: int) -> list[ExchangeOp]:
    """The chunk list libtffft executes for ``rank`` (host-only, no GPU)."""
    L = _lib.lib()
    n = ctypes.c_int64()
    _lib.check(L.tffft_exchange_schedule(n0, n1, n2, p, rank, None, 0, ctypes.byref(n)))
    buf = (ctypes.c_int64 * max(4 * n.value, 1))()
    _lib.check(L.tffft_exchange_schedule(n0, n1, n2, p, rank, buf, n.value, ctypes.byref(n)))
    return [ExchangeOp(*buf[4 * i: 4 * i + 4]) for i in range(n.value)]
