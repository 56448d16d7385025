"""Communicators for the GPU exchange (mirror of slabfft.transport's public
surface, reference pkg/src/slabfft/transport.py:35-43, 425-468).

Three transports behind one ``Endpoint``:

LOCAL   p endpoints share an in-process fabric on ONE device; each rank is
        driven by its own host thread (the reference's run_spmd model,
        transport.py:433-468).  The exchange is a device-side pull of every
        peer's staging band into this rank's landing buffer.
NCCL    one GPU per rank over NVLink/NVSwitch: one process per GPU (torchrun,
        ``init_nccl_endpoint``) or one process driving all of them
        (``make_communicators(p, devices=[...])``, ncclCommInitAll, one host
        thread per rank).  Grouped ncclSend/ncclRecv (PAIRWISE) or one
        ncclAlltoAll (COLLECTIVE) from the staging bands into the landing bands.
IPC     one process per rank, any device assignment (several processes may
        share a GPU): the plan's staging / landing buffers and events are
        exchanged as CUDA IPC handles; the exchange is the LOCAL fabric's pull
        across processes, with a torch.distributed (gloo) group as the host
        barrier (``init_ipc_endpoint``).
In every transport the FFT stage after the exchange reads the landing bands
through the STRIDED_INPLACE addressing: no unpack pass.
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass
from enum import Enum

import torch

from . import _lib
from .errors import ConfigurationError, TransportError

__all__ = [
    "CommMode",
    "CommPattern",
    "CopyCounter",
    "Endpoint",
    "make_communicators",
    "run_spmd",
    "init_nccl_endpoint",
    "nccl_loopback",
    "init_ipc_endpoint",
    "allgather_handles",
]


class CommMode(Enum):
    """Rank execution mode (transport.py:46-48).  On the GPU both run one
    host thread per rank; SERIAL is accepted for API parity."""

    THREADED = "threaded"
    SERIAL = "serial"


class CommPattern(Enum):
    PAIRWISE = "pairwise"
    COLLECTIVE = "collective"


@dataclass
class CopyCounter:
    """Bytes moved by the three kinds of copy pass (transport.py:97-114)."""

    bytes_packed: int = 0
    bytes_wire: int = 0
    bytes_unpacked: int = 0

    def reset(self) -> None:
        self.bytes_packed = self.bytes_wire = self.bytes_unpacked = 0

    def total(self) -> int:
        return self.bytes_packed + self.bytes_wire + self.bytes_unpacked

    def snapshot(self) -> tuple[int, int, int]:
        return (self.bytes_packed, self.bytes_wire, self.bytes_unpacked)


class Endpoint:
    """One rank's handle on the exchange fabric."""

    def __init__(self, handle: int, rank: int, p: int, device: int, kind: str,
                 host_barrier: threading.Barrier | None = None, group=None, keepalive=None):
        self._handle = ctypes.c_void_p(handle)
        self.rank = rank
        self.p = p
        self.device = device
        self.kind = kind
        self._host_barrier = host_barrier
        self._group = group            # torch.distributed group of an IPC endpoint
        self._keepalive = keepalive    # the ctypes barrier callback of an IPC endpoint
        self._closed = False

    @property
    def handle(self) -> ctypes.c_void_p:
        if self._closed:
            raise TransportError("endpoint is closed")
        return self._handle

    def barrier(self) -> None:
        """Device-complete barrier: drain this rank's stream, then meet the peers."""
        torch.cuda.current_stream(self.device).synchronize()
        if self.kind == "local":
            if self._host_barrier is not None:
                try:
                    self._host_barrier.wait(timeout=600)
                except threading.BrokenBarrierError as exc:
                    raise TransportError("fabric aborted while waiting at barrier") from exc
        elif self.kind == "ipc" and self.p > 1:
            torch.distributed.barrier(group=self._group)
        elif self.p > 1 and torch.distributed.is_initialized():
            torch.distributed.barrier()

    def allgather_bytes(self, blob: bytes) -> bytes:
        """Every rank's equal-sized blob, concatenated in rank order (the
        CUDA IPC handle exchange of NCCL peer-store and IPC plans)."""
        if self.kind == "ipc":
            return _allgather(blob, self.rank, self.p, self._group)
        return allgather_handles(blob, self.rank, self.p)

    def check(self) -> None:
        """Raise TransportError if the communicator failed asynchronously
        (NCCL: ncclCommGetAsyncError); a no-op for the local fabric."""
        _lib.check(_lib.lib().tffft_comm_check(self.handle))

    def abort(self) -> None:
        if self._host_barrier is not None:
            self._host_barrier.abort()
        _lib.check(_lib.lib().tffft_comm_abort(self._handle))

    def close(self) -> None:
        if not self._closed:
            _lib.lib().tffft_comm_destroy(self._handle)
            self._closed = True


def make_communicators(p: int, mode: CommMode = CommMode.THREADED, device: int | None = None,
                       timeout: float = 600.0, devices: list[int] | None = None) -> list[Endpoint]:
    """p connected endpoints (transport.py:425-430): sharing one in-process
    fabric on one GPU, or -- with ``devices`` (one distinct GPU per rank) --
    NCCL communicators created together by this process (ncclCommInitAll)."""
    if p < 1:
        raise ConfigurationError(f"communicator group needs p >= 1, got {p}")
    if devices is not None:
        devs = [int(d) for d in devices]
        if len(devs) != p:
            raise ConfigurationError(f"need {p} devices, got {len(devs)}")
        arr = (ctypes.c_void_p * p)()
        _lib.check(_lib.lib().tffft_comm_init_all(p, (ctypes.c_int * p)(*devs), arr))
        return [Endpoint(arr[r], r, p, devs[r], "nccl") for r in range(p)]
    dev = torch.cuda.current_device() if device is None else int(device)
    arr = (ctypes.c_void_p * p)()
    _lib.check(_lib.lib().tffft_comm_init_local(p, dev, arr))
    bar = threading.Barrier(p)
    return [Endpoint(arr[r], r, p, dev, "local", bar) for r in range(p)]


def run_spmd(p: int, fn, mode: CommMode = CommMode.THREADED, device: int | None = None,
             timeout: float = 600.0, devices: list[int] | None = None) -> list:
    """Run fn(endpoint) on p ranks (one host thread each) and return the
    results in rank order; the first failure aborts the fabric and is
    re-raised (transport.py:433-468).  ``devices``: one GPU per rank (NCCL)."""
    eps = make_communicators(p, mode, device, timeout, devices=devices)
    results: list = [None] * p
    errors: list[BaseException | None] = [None] * p

    def body(rank: int) -> None:
        try:
            torch.cuda.set_device(eps[rank].device)
            results[rank] = fn(eps[rank])
        except BaseException as exc:  # noqa: BLE001 - re-raised below
            errors[rank] = exc
            eps[rank].abort()

    threads = [threading.Thread(target=body, args=(r,), name=f"rank{r}") for r in range(p)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for ep in eps:
        ep.close()
    primary = next((e for e in errors if e is not None and not isinstance(e, TransportError)), None)
    if primary is None:
        primary = next((e for e in errors if e is not None), None)
    if primary is not None:
        raise primary
    return results


def nccl_loopback(device: int = 0, count: int = 1 << 20, dtype: str = "float64") -> bool:
    """Run the exchange's NCCL calls as a one-rank loopback on ``device``
    (``tffft_nccl_loopback``): grouped send/recv to self, all-to-all, the
    one-int all-reduce barrier.  Returns whether the loaded NCCL had
    ``ncclAlltoAll``; raises ``TransportError`` when a call or the payload
    comparison fails."""
    ran = ctypes.c_int(0)
    _lib.check(_lib.lib().tffft_nccl_loopback(int(device), int(count), 0 if dtype == "float64" else 1,
                                              ctypes.byref(ran)))
    return bool(ran.value)


def init_nccl_endpoint(device: int | None = None) -> Endpoint:
    """Endpoint for this process of a torch.distributed job (torchrun): the
    NCCL unique id is created on rank 0 and broadcast through the default
    process group (gloo or nccl)."""
    import torch.distributed as dist

    if not dist.is_initialized():
        raise ConfigurationError("torch.distributed is not initialised")
    rank, p = dist.get_rank(), dist.get_world_size()
    dev = torch.cuda.current_device() if device is None else int(device)
    uid = bytearray(128)
    if p > 1:
        if rank == 0:
            buf = ctypes.create_string_buffer(128)
            _lib.check(_lib.lib().tffft_get_unique_id(buf))
            uid = bytearray(buf.raw)
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0)
        uid = bytearray(obj[0])
    h = ctypes.c_void_p()
    _lib.check(_lib.lib().tffft_comm_init_rank(p, rank, bytes(uid), dev, ctypes.byref(h)))
    return Endpoint(h.value, rank, p, dev, "nccl")


def init_ipc_endpoint(device: int | None = None, group=None) -> Endpoint:
    """Endpoint for this process of a torch.distributed job whose exchange runs
    over CUDA IPC (any backend for ``group``, gloo included): the group's
    barrier is the library's host barrier, and plans all-gather their IPC
    handles over it.  Ranks may share a GPU."""
    import torch.distributed as dist

    if not dist.is_initialized():
        raise ConfigurationError("torch.distributed is not initialised")
    rank, p = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.cuda.current_device() if device is None else int(device)

    def _barrier(_ctx) -> int:
        try:
            dist.barrier(group=group)
            return 0
        except Exception:  # noqa: BLE001 - reported to the library as a transport failure
            return 1

    cb = _lib.BARRIER_FN(_barrier)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib().tffft_comm_init_ipc(p, rank, dev, ctypes.cast(cb, ctypes.c_void_p), None,
                                              ctypes.byref(h)))
    return Endpoint(h.value, rank, p, dev, "ipc", group=group, keepalive=cb)


def _allgather(blob: bytes, rank: int, p: int, group) -> bytes:
    import torch.distributed as dist

    got: list = [None] * p
    dist.all_gather_object(got, bytes(blob), group=group)
    if {len(b) for b in got} != {len(blob)}:
        raise TransportError(f"handle sizes differ across ranks: {sorted({len(b) for b in got})}")
    return b"".join(got)


def allgather_handles(handle: bytes, rank: int, p: int) -> bytes:
    """All-gather one fixed-size handle per rank over the default
    torch.distributed group and return the concatenation in RANK order (the
    layout tffft_plan_attach_peers expects).  Every rank must call it."""
    import torch.distributed as dist

    if not dist.is_initialized():
        raise ConfigurationError("torch.distributed is not initialised")
    if dist.get_world_size() != p or dist.get_rank() != rank:
        raise ConfigurationError(f"process group (rank {dist.get_rank()} of {dist.get_world_size()}) does not match "
                                 f"the communicator (rank {rank} of {p})")
    got: list = [None] * p
    dist.all_gather_object(got, bytes(handle))
    sizes = {len(h) for h in got}
    if sizes != {len(handle)}:
        raise TransportError(f"handle sizes differ across ranks: {sorted(sizes)}")
    return b"".join(got)
