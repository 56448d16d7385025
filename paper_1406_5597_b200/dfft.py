"""Distributed 3D real FFT, B200 path: plan / forward (r2c) / inverse (c2r)
(mirror of slabfft.dfft, reference pkg/src/slabfft/dfft.py:52-270).

``plan(grid, comm, Strategy.STRIDED)`` builds a per-rank libtffft plan;
``forward`` returns a STRIDED_INPLACE ``SpectralSlab`` backed by plan-owned
device memory (valid until the next call, dfft.py:152-153) and ``inverse``
consumes its spectral input and returns a plan-owned ``RealSlab``
normalised by 1/(n0 n1 n2) (dfft.py:179-215).  All transform arithmetic runs
in the sm_100a kernels of libtffft.so; there is no CPU path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import ConfigurationError, ContractError, ProtocolError
from .exchange import Strategy
from .layout import DistAxis, GlobalGrid, RealSlab, SlabLayout, SpectralSlab, SpectralTag, validate
from .transport import CommPattern, CopyCounter, Endpoint

__all__ = ["FftPlan", "plan", "forward", "inverse", "forward_many", "inverse_many", "gather_spectral",
           "scatter_real", "gather_real", "scatter_spectral", "DTYPES"]

# precision name -> (C enum, real torch dtype, complex torch dtype)
DTYPES = {
    "float64": (0, torch.float64, torch.complex128),
    "float32": (1, torch.float32, torch.complex64),
}


@dataclass
class FftPlan:
    """Everything one rank needs to run GPU forward/inverse transforms (dfft.py:55-90)."""

    grid: GlobalGrid
    comm: Endpoint
    strategy: Strategy
    comm_pattern: CommPattern
    real_layout: SlabLayout
    spectral_layout: SlabLayout
    dtype: str
    handle: ctypes.c_void_p
    work1: torch.Tensor      # spectral slab(s), plan-owned (forward output); batch slabs back to back
    real_out: torch.Tensor   # real slab(s), plan-owned (inverse output); batch slabs back to back
    check_consistency: bool = True
    batch: int = 1
    last_imag_residue: float = 0.0
    _timing: bool = field(default=False, repr=False)

    @property
    def p(self) -> int:
        return self.comm.p

    @property
    def rank(self) -> int:
        return self.comm.rank

    @property
    def device(self) -> torch.device:
        return torch.device("cuda", self.comm.device)

    @property
    def counters(self) -> CopyCounter:
        b = (ctypes.c_uint64 * 3)()
        _lib.check(_lib.lib().tffft_counters(self.handle, b))
        return CopyCounter(int(b[0]), int(b[1]), int(b[2]))

    @property
    def timers_us(self) -> dict:
        """Per-stage device times (CUDA events) since the last reset; enable
        with ``enable_timing()``.  Synchronises on the recorded events."""
        ms = (ctypes.c_double * 3)()
        _lib.check(_lib.lib().tffft_stage_times(self.handle, ms))
        return {"stage1_us": ms[0] * 1e3, "exchange_us": ms[1] * 1e3, "stage3_us": ms[2] * 1e3}

    def enable_timing(self, on: bool = True) -> None:
        _lib.check(_lib.lib().tffft_set_timing(self.handle, int(on)))
        self._timing = on

    def reset_instrumentation(self) -> None:
        _lib.check(_lib.lib().tffft_reset_instrumentation(self.handle))
        self.last_imag_residue = 0.0

    @property
    def launches(self) -> int:
        n = ctypes.c_uint64()
        _lib.check(_lib.lib().tffft_launch_count(self.handle, ctypes.byref(n)))
        return int(n.value)

    @property
    def algorithms(self) -> tuple[str, ...]:
        f = ctypes.c_int()
        _lib.check(_lib.lib().tffft_plan_flags(self.handle, ctypes.byref(f)))
        return tuple(a for a, bit in ALGORITHM_FLAGS.items() if f.value & bit)

    @property
    def workspace_bytes(self) -> int:
        n = ctypes.c_size_t()
        _lib.check(_lib.lib().tffft_plan_workspace_bytes(self.handle, ctypes.byref(n)))
        return int(n.value)

    def set_check_consistency(self, mode: bool | str) -> None:
        """Switch the Hermitian check between True (per call, synchronous),
        False and "deferred" (device-side, see collect_consistency)."""
        if mode not in (True, False, "deferred"):
            raise ConfigurationError(f"check_consistency must be True, False or 'deferred', got {mode!r}")
        with torch.cuda.device(self.comm.device):
            _lib.check(_lib.lib().tffft_set_consistency_mode(self.handle, int(mode == "deferred")))
        self.check_consistency = mode

    def collect_consistency(self) -> int:
        """Deferred consistency mode (``check_consistency="deferred"``):
        synchronise, and raise ConsistencyError if any inverse since the last
        collect had a non-Hermitian half spectrum (kernels.py:225-238).
        Returns the number of inverse calls checked."""
        res = ctypes.c_double()
        calls = ctypes.c_uint64()
        status = _lib.lib().tffft_consistency_collect(self.handle, ctypes.byref(res), ctypes.byref(calls))
        self.last_imag_residue = max(self.last_imag_residue, float(res.value))
        _lib.check(status)
        return int(calls.value)

    def poison(self) -> None:
        """Debug: fill the plan's exchange buffers and row records with NaN
        (tffft_plan_poison); a stage reading an element no stage wrote then
        yields NaN.  Synchronous."""
        _lib.check(_lib.lib().tffft_plan_poison(self.handle))

    def close(self) -> None:
        if self.handle:
            _lib.lib().tffft_plan_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


ALGORITHM_FLAGS = {"fused_stage1": 1, "fourstep_stage3": 2, "peer_stores": 8, "tma_columns": 16,
                   "chunked_exchange": 32}
TRANSPOSE_FLAG = 4


_PATTERN_CODE = {CommPattern.PAIRWISE: 0, CommPattern.COLLECTIVE: 1}  # TFFFT_PAIRWISE / TFFFT_COLLECTIVE


def _spectral_tag(strategy: Strategy) -> SpectralTag:
    return SpectralTag.STRIDED_INPLACE if strategy is Strategy.STRIDED else SpectralTag.CONTIGUOUS_FLIPPED


def plan(grid: GlobalGrid, comm: Endpoint, strategy: Strategy = Strategy.STRIDED,
         comm_pattern: CommPattern = CommPattern.PAIRWISE, dtype: str = "float64",
         check_consistency: bool | str = True, algorithms: tuple[str, ...] | None = None,
         batch: int = 1) -> FftPlan:
    """Per-rank plan (dfft.py:93-145).  Collective on a LOCAL fabric, and on
    NCCL (peer stores) / IPC communicators, whose buffers are exchanged here.

    ``algorithms`` selects optional kernel schedules ("fused_stage1",
    "fourstep_stage3", "peer_stores", "tma_columns", "chunked_exchange");
    None takes the library
    defaults (TFFFT_FUSE / TFFFT_FOURSTEP / TFFFT_TMA_COLS / TFFFT_WPC
    environment switches; by default the 512-, 1024- and 2048-point column
    passes are TMA-fed at any p: the warp-per-column kernels or
    col_tma_kernel).  ``batch`` > 1 makes a batched plan: ``forward_many`` /
    ``inverse_many`` transform ``batch`` fields per call (one launch per stage
    over all fields at p = 1; field c's exchange overlapping field c+1's
    compute at p > 1)."""
    validate(grid, comm.p)
    if check_consistency not in (True, False, "deferred"):
        raise ConfigurationError(f"check_consistency must be True, False or 'deferred', got {check_consistency!r}")
    if not isinstance(batch, int) or batch < 1:
        raise ConfigurationError(f"batch must be a positive int, got {batch!r}")
    if not isinstance(comm_pattern, CommPattern):
        raise ConfigurationError(f"comm_pattern must be a CommPattern, got {comm_pattern!r}")
    if dtype not in DTYPES:
        raise ConfigurationError(f"dtype must be one of {sorted(DTYPES)}, got {dtype!r}")
    code, rdt, cdt = DTYPES[dtype]
    flags = -1
    if algorithms is not None:
        unknown = set(algorithms) - set(ALGORITHM_FLAGS)
        if unknown:
            raise ConfigurationError(f"unknown algorithms {sorted(unknown)}; choose from {sorted(ALGORITHM_FLAGS)}")
        flags = sum(ALGORITHM_FLAGS[a] for a in set(algorithms))
    if strategy is Strategy.TRANSPOSE:  # the paper's baseline: pack, contiguous exchange, unpack
        flags = (0 if flags < 0 else flags) | TRANSPOSE_FLAG
    h = ctypes.c_void_p()
    with torch.cuda.device(comm.device):
        _lib.check(_lib.lib().tffft_plan_create_batched(grid.n0, grid.n1, grid.n2, code, _PATTERN_CODE[comm_pattern],
                                                        flags, batch, comm.handle, ctypes.byref(h)))
        p, rank = comm.p, comm.rank
        dev = torch.device("cuda", comm.device)
        work1 = torch.empty(batch * (grid.n0 // p) * grid.n1 * grid.n2c, dtype=cdt, device=dev)
        real_out = torch.empty(batch * (grid.n0 // p) * grid.n1 * grid.n2, dtype=rdt, device=dev)
    if check_consistency == "deferred":  # every inverse folds its check on the device
        with torch.cuda.device(comm.device):
            _lib.check(_lib.lib().tffft_set_consistency_mode(h, 1))
    peer_stores = flags >= 0 and bool(flags & ALGORITHM_FLAGS["peer_stores"])
    if comm.p > 1 and (comm.kind == "ipc" or (comm.kind == "nccl" and peer_stores)):
        # CUDA IPC: every rank exports its exchange buffers (and, on an IPC
        # communicator, its events); the blobs are all-gathered in rank order
        # and each rank maps the peers' (fused exchange over NVLink for NCCL)
        n = ctypes.c_size_t()
        _lib.check(_lib.lib().tffft_plan_ipc_blob_bytes(h, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        with torch.cuda.device(comm.device):
            _lib.check(_lib.lib().tffft_plan_ipc_export(h, buf))
        allh = comm.allgather_bytes(buf.raw)
        with torch.cuda.device(comm.device):
            _lib.check(_lib.lib().tffft_plan_ipc_attach(h, allh))
    return FftPlan(
        grid=grid, comm=comm, strategy=strategy, comm_pattern=comm_pattern,
        real_layout=SlabLayout(grid, p, rank, DistAxis.REAL_AXIS0),
        spectral_layout=SlabLayout(grid, p, rank, DistAxis.SPECTRAL_AXIS1),
        dtype=dtype, handle=h, work1=work1, real_out=real_out,
        check_consistency=check_consistency, batch=batch,
    )


def _check_tensor(t: torch.Tensor, fp: FftPlan, want: torch.dtype, what: str) -> None:
    if t.dtype != want:
        raise ContractError(f"{what} must be {want} for a {fp.dtype} plan, got {t.dtype}")
    if t.device != fp.device:
        raise ContractError(f"{what} must live on {fp.device}, got {t.device}")
    if not t.is_contiguous():
        raise ContractError(f"{what} must be contiguous")


def _stream(fp: FftPlan) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(fp.device).cuda_stream)


def forward(fp: FftPlan, real: RealSlab, out: torch.Tensor | None = None) -> SpectralSlab:
    """Distributed forward r2c of this rank's slab (dfft.py:148-176).

    Collective.  Logical element (j, r, k) of the result is bin
    (r, rank*(n1/p)+j, k) of the unnormalised global spectrum, stored
    STRIDED_INPLACE (Strategy.STRIDED) or CONTIGUOUS_FLIPPED
    (Strategy.TRANSPOSE).  The result is backed by plan memory unless ``out``
    is given."""
    if fp.batch != 1:
        raise ContractError(f"plan has batch={fp.batch}: use forward_many")
    if real.layout != fp.real_layout:
        raise ContractError(f"slab layout {real.layout} does not match plan {fp.real_layout}")
    _, rdt, cdt = DTYPES[fp.dtype]
    _check_tensor(real.data, fp, rdt, "real slab")
    dst = fp.work1 if out is None else out
    _check_tensor(dst, fp, cdt, "spectral output")
    if dst.numel() != fp.work1.numel():
        raise ContractError(f"spectral output needs {fp.work1.numel()} elements, got {dst.numel()}")
    _lib.check(_lib.lib().tffft_forward(fp.handle, ctypes.c_void_p(real.data.data_ptr()),
                                        ctypes.c_void_p(dst.data_ptr()), _stream(fp)))
    return SpectralSlab(fp.spectral_layout, _spectral_tag(fp.strategy), dst)


def inverse(fp: FftPlan, spec: SpectralSlab, out: torch.Tensor | None = None) -> RealSlab:
    """Distributed inverse c2r normalised by 1/(n0 n1 n2) (dfft.py:179-215).

    Collective; consumes ``spec`` in place.  With ``fp.check_consistency``
    True the call synchronises and raises ConsistencyError for a non-Hermitian
    half spectrum, as the reference's _c2r_rows does (kernels.py:223-238);
    with "deferred" the same check runs on the device and is reported by
    ``fp.collect_consistency()``."""
    if fp.batch != 1:
        raise ContractError(f"plan has batch={fp.batch}: use inverse_many")
    expected = _spectral_tag(fp.strategy)
    if spec.tag is not expected:
        raise ContractError(f"plan strategy {fp.strategy} expects a {expected} slab, got {spec.tag}")
    if spec.layout != fp.spectral_layout:
        raise ContractError(f"slab layout {spec.layout} does not match plan")
    _, rdt, cdt = DTYPES[fp.dtype]
    _check_tensor(spec.data, fp, cdt, "spectral slab")
    dst = fp.real_out if out is None else out
    _check_tensor(dst, fp, rdt, "real output")
    if dst.numel() != fp.real_out.numel():
        raise ContractError(f"real output needs {fp.real_out.numel()} elements, got {dst.numel()}")
    _lib.check(_lib.lib().tffft_inverse(fp.handle, ctypes.c_void_p(spec.data.data_ptr()),
                                        ctypes.c_void_p(dst.data_ptr()), _stream(fp)))
    if fp.check_consistency is True:
        _check_consistency(fp)
    return RealSlab(fp.real_layout, dst)


def _check_consistency(fp: FftPlan) -> None:
    res = ctypes.c_double()
    status = _lib.lib().tffft_consistency(fp.handle, ctypes.byref(res))
    fp.last_imag_residue = max(fp.last_imag_residue, float(res.value))
    _lib.check(status)


def forward_many(fp: FftPlan, real: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Forward r2c of ``fp.batch`` fields in one call (batched plan).

    ``real`` holds the fields' real slabs back to back (``batch`` x
    n0/p*n1*n2 elements, e.g. a (batch, slab) tensor); returns their
    STRIDED_INPLACE spectral slabs back to back (plan memory unless ``out``)."""
    _, rdt, cdt = DTYPES[fp.dtype]
    if fp.strategy is not Strategy.STRIDED:
        raise ContractError("forward_many runs the STRIDED strategy")
    _check_tensor(real, fp, rdt, "real slabs")
    if real.numel() != fp.real_out.numel():
        raise ContractError(f"real slabs need {fp.real_out.numel()} elements ({fp.batch} fields), got {real.numel()}")
    dst = fp.work1 if out is None else out
    _check_tensor(dst, fp, cdt, "spectral output")
    if dst.numel() != fp.work1.numel():
        raise ContractError(f"spectral output needs {fp.work1.numel()} elements, got {dst.numel()}")
    _lib.check(_lib.lib().tffft_forward(fp.handle, ctypes.c_void_p(real.data_ptr()),
                                        ctypes.c_void_p(dst.data_ptr()), _stream(fp)))
    return dst


def inverse_many(fp: FftPlan, spec: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Inverse c2r of ``fp.batch`` fields in one call (batched plan); consumes
    ``spec`` (the fields' spectral slabs back to back).  The Hermitian
    consistency check runs once for the whole batch."""
    _, rdt, cdt = DTYPES[fp.dtype]
    if fp.strategy is not Strategy.STRIDED:
        raise ContractError("inverse_many runs the STRIDED strategy")
    _check_tensor(spec, fp, cdt, "spectral slabs")
    if spec.numel() != fp.work1.numel():
        raise ContractError(f"spectral slabs need {fp.work1.numel()} elements ({fp.batch} fields), got {spec.numel()}")
    dst = fp.real_out if out is None else out
    _check_tensor(dst, fp, rdt, "real output")
    if dst.numel() != fp.real_out.numel():
        raise ContractError(f"real output needs {fp.real_out.numel()} elements, got {dst.numel()}")
    _lib.check(_lib.lib().tffft_inverse(fp.handle, ctypes.c_void_p(spec.data_ptr()),
                                        ctypes.c_void_p(dst.data_ptr()), _stream(fp)))
    if fp.check_consistency is True:
        _check_consistency(fp)
    return dst


# ---------------------------------------------------------------------------
# host-side helpers (dfft.py:218-270), torch or numpy in, torch/numpy out
# ---------------------------------------------------------------------------

def _np(t) -> np.ndarray:
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


def scatter_real(values, grid: GlobalGrid, p: int, device=None, dtype: str = "float64") -> list[RealSlab]:
    """Split a global real field into the p axis-0 slabs on ``device``."""
    if dtype not in DTYPES:
        raise ConfigurationError(f"dtype must be one of {sorted(DTYPES)}")
    rdt = DTYPES[dtype][1]
    vals = values if isinstance(values, torch.Tensor) else torch.from_numpy(np.asarray(values, dtype=np.float64))
    if tuple(vals.shape) != (grid.n0, grid.n1, grid.n2):
        raise ContractError(f"field shape {tuple(vals.shape)} does not match grid {grid}")
    validate(grid, p)
    n0p = grid.n0 // p
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    return [RealSlab(SlabLayout(grid, p, r, DistAxis.REAL_AXIS0),
                     vals[r * n0p:(r + 1) * n0p].to(device=dev, dtype=rdt).contiguous().reshape(-1))
            for r in range(p)]


def gather_real(slabs: list[RealSlab]) -> np.ndarray:
    """Reassemble the global real field (numpy) from the p axis-0 slabs."""
    if not slabs:
        raise ProtocolError("no slabs to gather")
    lay0 = slabs[0].layout
    p, g = lay0.p, lay0.grid
    ranks = sorted(s.layout.rank for s in slabs)
    if len(slabs) != p or ranks != list(range(p)):
        raise ProtocolError(f"need one slab per rank 0..{p - 1}, got ranks {ranks}")
    out = np.empty((g.n0, g.n1, g.n2), dtype=_np(slabs[0].data).dtype)
    for s in slabs:
        r = s.layout.rank
        out[r * lay0.n0p:(r + 1) * lay0.n0p] = _np(s.data).reshape(lay0.n0p, g.n1, g.n2)
    return out


def gather_spectral(slabs: list[SpectralSlab]) -> np.ndarray:
    """Global (n0, n1, n2c) spectrum (numpy) from all ranks' slabs (dfft.py:218-238)."""
    if not slabs:
        raise ProtocolError("no slabs to gather")
    lay0 = slabs[0].layout
    p, g = lay0.p, lay0.grid
    ranks = sorted(s.layout.rank for s in slabs)
    if len(slabs) != p or ranks != list(range(p)):
        raise ProtocolError(f"need one slab per rank 0..{p - 1}, got ranks {ranks}")
    n1p = lay0.n1p
    out = np.empty((g.n0, g.n1, g.n2c), dtype=_np(slabs[0].data).dtype)
    for s in slabs:
        q = s.layout.rank
        out[:, q * n1p:(q + 1) * n1p, :] = _np(s.as_logical()).transpose(1, 0, 2)
    return out


def scatter_spectral(glob, grid: GlobalGrid, p: int, device=None, dtype: str = "float64") -> list[SpectralSlab]:
    """Inverse of gather_spectral: each rank's STRIDED_INPLACE slab on ``device``."""
    cdt = DTYPES[dtype][2]
    g = torch.as_tensor(glob)
    if tuple(g.shape) != (grid.n0, grid.n1, grid.n2c):
        raise ContractError(f"spectrum shape {tuple(g.shape)} does not match grid {grid}")
    validate(grid, p)
    n0p, n1p = grid.n0 // p, grid.n1 // p
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    out = []
    for q in range(p):
        band = g[:, q * n1p:(q + 1) * n1p, :].reshape(p, n0p, n1p, grid.n2c).permute(1, 0, 2, 3)
        out.append(SpectralSlab(SlabLayout(grid, p, q, DistAxis.SPECTRAL_AXIS1), SpectralTag.STRIDED_INPLACE,
                                band.to(device=dev, dtype=cdt).contiguous().reshape(-1)))
    return out
