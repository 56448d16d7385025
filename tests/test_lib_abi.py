"""The C-ABI library: loads without a GPU, exports every symbol
include/tffft.h declares, and its host-only entry points (exchange
schedule, radix schedule, communicator bookkeeping, argument checking)."""

import ctypes
import os
import re

import pytest

import paper_1406_5597_b200 as tf
from paper_1406_5597_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "tffft.h")).read()
    return sorted(set(re.findall(r"\b(tffft_\w+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SYMBOLS)


def test_version():
    assert _lib.lib().tffft_version() >= 100


def test_radix_schedule_matches_design():
    lib = _lib.lib()
    got = {}
    for L in range(0, 13):
        r = (ctypes.c_int * 8)()
        n = ctypes.c_int()
        _lib.check(lib.tffft_radix_schedule(L, r, ctypes.byref(n)))
        got[L] = [r[i] for i in range(n.value)]
        prod = 1
        for x in got[L]:
            prod *= x
            assert x <= (32 if L in (9, 10) else 16)
        assert prod == 1 << L
    # 512- and 1024-point transforms (the headline rows and columns) run as two
    # radix-32/16 passes: one shared-memory exchange instead of two
    assert got[10] == [32, 32] and got[9] == [32, 16] and got[11] == [16, 16, 8]


@pytest.mark.parametrize("n0,n1,n2,p", [(4, 4, 2, 2), (8, 8, 8, 4), (16, 8, 32, 8), (128, 128, 128, 2)])
def test_exchange_schedule_geometry(n0, n1, n2, p):
    """One send of staging band q and one receive into landing band q per peer
    (the reference posts one strided LayoutDescriptor per peer, exchange.py:114-119);
    every off-rank band is sent and received exactly once."""
    n0p, n1p, n2c = n0 // p, n1 // p, n2 // 2 + 1
    band = n0p * n1p * n2c
    for rank in range(p):
        ops = tf.exchange_schedule(n0, n1, n2, p, rank)
        assert len(ops) == p - 1
        assert sorted(op.peer for op in ops) == [q for q in range(p) if q != rank]
        for op in ops:
            assert op.count == band
            assert op.send_offset == op.peer * band and op.recv_offset == op.peer * band


def test_exchange_schedule_rejects_bad_geometry():
    with pytest.raises(tf.ConfigurationError):
        tf.exchange_schedule(6, 8, 8, 4, 0)


def test_local_communicators_host_bookkeeping():
    lib = _lib.lib()
    arr = (ctypes.c_void_p * 3)()
    _lib.check(lib.tffft_comm_init_local(3, 0, arr))
    for r in range(3):
        v = ctypes.c_int()
        _lib.check(lib.tffft_comm_rank(arr[r], ctypes.byref(v)))
        assert v.value == r
        _lib.check(lib.tffft_comm_size(arr[r], ctypes.byref(v)))
        assert v.value == 3
    _lib.check(lib.tffft_comm_abort(arr[0]))
    for r in range(3):
        _lib.check(lib.tffft_comm_destroy(arr[r]))


def test_plan_create_validates_before_touching_the_gpu():
    lib = _lib.lib()
    arr = (ctypes.c_void_p * 2)()
    _lib.check(lib.tffft_comm_init_local(2, 0, arr))
    h = ctypes.c_void_p()
    cases = [((6, 8, 8), tf.ConfigurationError),   # not a power of two
             ((8, 8, 1), tf.ConfigurationError),   # axis < 2
             ((8, 8, 8192), tf.SizeError),         # beyond the kernels' 4096 limit
             ((8, 6, 8), tf.ConfigurationError)]
    for (n0, n1, n2), err in cases:
        with pytest.raises(err):
            _lib.check(lib.tffft_plan_create(n0, n1, n2, 0, 0, arr[0], ctypes.byref(h)))
    with pytest.raises(tf.ConfigurationError):  # unknown dtype
        _lib.check(lib.tffft_plan_create(8, 8, 8, 7, 0, arr[0], ctypes.byref(h)))
    with pytest.raises(tf.ConfigurationError):  # unknown comm pattern
        _lib.check(lib.tffft_plan_create(8, 8, 8, 0, 7, arr[0], ctypes.byref(h)))
    for r in range(2):
        lib.tffft_comm_destroy(arr[r])


def test_status_codes_map_to_reference_exceptions():
    from paper_1406_5597_b200.errors import STATUS_TO_ERROR
    assert STATUS_TO_ERROR[1] is tf.SizeError
    assert STATUS_TO_ERROR[3] is tf.ConfigurationError
    assert STATUS_TO_ERROR[4] is tf.ContractError
    assert STATUS_TO_ERROR[7] is tf.ConsistencyError
    assert issubclass(tf.ConfigurationError, ValueError) and issubclass(tf.ContractError, tf.SlabFftError)


def test_comm_check_local_fabric_is_healthy():
    """tffft_comm_check (SURVEY §5 failure detection) on the local fabric:
    nothing asynchronous can fail, the call returns TFFFT_OK; a null
    communicator is a ConfigurationError."""
    import paper_1406_5597_b200 as tf
    lib = _lib.lib()
    arr = (ctypes.c_void_p * 2)()
    _lib.check(lib.tffft_comm_init_local(2, 0, arr))
    try:
        for r in range(2):
            assert lib.tffft_comm_check(arr[r]) == 0
        with pytest.raises(tf.ConfigurationError):
            _lib.check(lib.tffft_comm_check(None))
    finally:
        for r in range(2):
            lib.tffft_comm_destroy(arr[r])


def test_round2_entry_points_validate_on_the_host():
    """Host-side argument checks of the round-2 C ABI (no GPU needed):
    comm_init_all refuses a device listed twice (NCCL needs one GPU per rank),
    plan_create_batched refuses batch < 1, comm_init_ipc needs a barrier,
    comm_barrier is refused on NCCL-kind communicators and passes on a p = 1
    local fabric, ipc export is refused on local-fabric plans."""
    lib = _lib.lib()
    comms = (ctypes.c_void_p * 2)()
    with pytest.raises(tf.ConfigurationError, match="listed twice"):
        _lib.check(lib.tffft_comm_init_all(2, (ctypes.c_int * 2)(0, 0), comms))
    one = (ctypes.c_void_p * 1)()
    _lib.check(lib.tffft_comm_init_all(1, (ctypes.c_int * 1)(0), one))  # p = 1: no NCCL needed
    with pytest.raises(tf.ConfigurationError):
        _lib.check(lib.tffft_comm_barrier(one[0]))
    lib.tffft_comm_destroy(one[0])
    arr = (ctypes.c_void_p * 1)()
    _lib.check(lib.tffft_comm_init_local(1, 0, arr))
    _lib.check(lib.tffft_comm_barrier(arr[0]))
    h = ctypes.c_void_p()
    with pytest.raises(tf.ConfigurationError, match="batch"):
        _lib.check(lib.tffft_plan_create_batched(8, 8, 8, 0, 0, 0, 0, arr[0], ctypes.byref(h)))
    with pytest.raises(tf.ConfigurationError):
        _lib.check(lib.tffft_plan_ipc_export(None, None))
    lib.tffft_comm_destroy(arr[0])
    ipc = ctypes.c_void_p()
    with pytest.raises(tf.ConfigurationError):
        _lib.check(lib.tffft_comm_init_ipc(2, 0, 0, None, None, ctypes.byref(ipc)))
    with pytest.raises(tf.ConfigurationError):
        _lib.check(lib.tffft_comm_init_ipc(2, 5, 0, ctypes.cast(_lib.BARRIER_FN(lambda c: 0), ctypes.c_void_p), None,
                                           ctypes.byref(ipc)))


def test_ipc_barrier_callback_failure_is_a_transport_error():
    """A failing host barrier (the callback returns non-zero) surfaces as
    TransportError, and the communicator stays aborted (transport.py:209-219)."""
    lib = _lib.lib()
    cb = _lib.BARRIER_FN(lambda ctx: 1)
    c = ctypes.c_void_p()
    _lib.check(lib.tffft_comm_init_ipc(2, 0, 0, ctypes.cast(cb, ctypes.c_void_p), None, ctypes.byref(c)))
    try:
        with pytest.raises(tf.TransportError):
            _lib.check(lib.tffft_comm_barrier(c))
        with pytest.raises(tf.TransportError, match="aborted"):
            _lib.check(lib.tffft_comm_barrier(c))
    finally:
        lib.tffft_comm_destroy(c)
