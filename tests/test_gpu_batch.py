"""Batched plans (plan_create(..., batch, ...)) and
single-process multi-device communicators (comm_init_all).

A batched plan transforms `batch` fields per call: at p = 1 each stage is one
launch over all fields, at p > 1 the fields run through a two-deep pipeline in
which field c's exchange overlaps field c+1's producing stage.  Every field
must equal the oracle's transform of that field (relative L2 <= 1e-12 /
1e-5), for both directions, every transport pattern and the peer-store
exchange.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_1406_5597_b200 as tf

pytestmark = pytest.mark.gpu
TOL = {"float64": 1e-12, "float32": 1e-5}


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def run_batched(fields, p, dtype="float64", pattern=tf.CommPattern.PAIRWISE, algorithms=None):
    """forward_many then inverse_many of len(fields) fields on p local-fabric
    ranks; per field: per-rank spectral buffers and the gathered real output."""
    shape = fields[0].shape
    grid = tf.GlobalGrid(*shape)
    B = len(fields)
    slabs = [tf.scatter_real(x, grid, p, dtype=dtype) for x in fields]

    def body(ep):
        fp = tf.plan(grid, ep, tf.Strategy.STRIDED, comm_pattern=pattern, dtype=dtype, batch=B,
                     algorithms=algorithms)
        real = torch.cat([slabs[c][ep.rank].data for c in range(B)])
        spec = tf.forward_many(fp, real)
        fwd = spec.view(B, -1).cpu().numpy().copy()
        launches = fp.launches
        back = tf.inverse_many(fp, spec)
        inv = back.view(B, -1).cpu().numpy().copy()
        fp.close()
        return fwd, inv, launches

    return tf.run_spmd(p, body)


@pytest.mark.parametrize("shape,p", [((64, 64, 64), 1), ((1024, 8, 16), 1), ((16, 1024, 8), 1),
                                     ((32, 64, 16), 2), ((64, 32, 8), 4), ((16, 16, 32), 8)],
                         ids=str)
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_batched_matches_oracle(shape, p, dtype):
    B = 3
    fields = [oracle.uniform_field(shape, seed=40 + c) for c in range(B)]
    if dtype == "float32":
        fields = [f.astype(np.float32).astype(np.float64) for f in fields]
    res = run_batched(fields, p, dtype)
    for c in range(B):
        ref = oracle.forward_all(fields[c], p)
        for q in range(p):
            assert rel(res[q][0][c], ref[q]) <= TOL[dtype], (c, q)
        back = np.concatenate([res[q][1][c] for q in range(p)]).reshape(shape)
        assert rel(back, fields[c]) <= TOL[dtype], c


def test_batched_p1_is_one_launch_per_stage():
    """p = 1: the three fields share every launch (six kernels per pair + the
    consistency reduction), not three times as many."""
    shape = (64, 64, 64)
    fields = [oracle.uniform_field(shape, seed=c) for c in range(3)]
    res = run_batched(fields, 1)
    assert res[0][2] == 3  # forward: r2c rows, n1 columns, n0 columns -- for all 3 fields


@pytest.mark.parametrize("pattern", [tf.CommPattern.PAIRWISE, tf.CommPattern.COLLECTIVE])
@pytest.mark.parametrize("algorithms", [None, ("peer_stores",)], ids=["pull", "peer_stores"])
def test_batched_pipeline_patterns(pattern, algorithms):
    """p > 1 pipeline with 5 fields (both buffer sets reused twice), both
    exchange patterns and the fused peer-store exchange."""
    shape, p, B = (32, 32, 16), 4, 5
    fields = [oracle.normal_field(shape, seed=70 + c) for c in range(B)]
    res = run_batched(fields, p, "float64", pattern, algorithms)
    for c in range(B):
        ref = oracle.forward_all(fields[c], p)
        for q in range(p):
            assert rel(res[q][0][c], ref[q]) <= 1e-12, (c, q)
        back = np.concatenate([res[q][1][c] for q in range(p)]).reshape(shape)
        assert rel(back, fields[c]) <= 1e-12, c


def test_batched_consistency_names_the_field():
    """The Hermitian check covers every field of the batch (kernels.py:225-238)."""
    shape = (8, 8, 8)
    grid = tf.GlobalGrid(*shape)
    ep = tf.make_communicators(1)[0]
    fp = tf.plan(grid, ep, batch=2)
    x = torch.cat([tf.scatter_real(oracle.uniform_field(shape, c), grid, 1)[0].data for c in range(2)])
    spec = tf.forward_many(fp, x)
    spec.view(2, 8, 8, 5)[1, 3, 2, 0] += 1j  # a DC bin of field 1 becomes non-real
    with pytest.raises(tf.ConsistencyError, match="field 1"):
        tf.inverse_many(fp, spec)
    fp.close()


def test_turbulence_batched_equals_unbatched():
    """BASELINE config 5 through a batched plan: the 3-component inverse ->
    forward round trip gives the same spectra as three single-field calls."""
    shape = (64, 64, 64)
    grid = tf.GlobalGrid(*shape)
    ep = tf.make_communicators(1)[0]
    fp1 = tf.plan(grid, ep)
    fp3 = tf.plan(grid, ep, batch=3)
    noise = torch.cat([tf.scatter_real(oracle.normal_field(shape, 5 + c), grid, 1)[0].data for c in range(3)])
    specs = tf.turbulence_spectra(fp3, noise, 1.0, 21.0).clone()
    singles = []
    for c in range(3):
        s = tf.turbulence_spectrum(fp1, tf.RealSlab(fp1.real_layout, noise.view(3, -1)[c]), 1.0, 21.0)
        singles.append(s.data.clone())
    for c in range(3):
        assert torch.equal(specs.view(3, -1)[c], singles[c])  # same kernels, same bits
    ref = specs.clone()
    reals = tf.inverse_batch(fp3, list(specs.view(3, -1)))
    out = tf.forward_batch(fp3, reals)
    for c in range(3):
        assert rel(out[c].data.cpu().numpy(), ref.view(3, -1)[c].cpu().numpy()) <= 1e-12
    fp1.close()
    fp3.close()


def test_comm_init_all_single_device():
    """ncclCommInitAll analogue (comm_init_all): one device per rank; a list
    naming one device twice is refused (NCCL needs distinct GPUs)."""
    shape = (32, 16, 8)
    x = oracle.uniform_field(shape, 1)
    grid = tf.GlobalGrid(*shape)
    ref = oracle.forward_all(x, 1)[0]

    def body(ep):
        assert ep.kind == "nccl" and ep.device == 0
        fp = tf.plan(grid, ep)
        out = tf.forward(fp, tf.scatter_real(x, grid, 1)[0]).data.cpu().numpy().copy()
        fp.close()
        return out

    got = tf.run_spmd(1, body, devices=[0])[0]
    assert rel(got, ref) <= 1e-12
    with pytest.raises(tf.ConfigurationError):
        tf.make_communicators(2, devices=[0, 0])


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("pattern", [tf.CommPattern.PAIRWISE, tf.CommPattern.COLLECTIVE])
@pytest.mark.parametrize("shape", [(1024, 64, 16), (32, 1024, 16)], ids=lambda v: "x".join(map(str, v)))
def test_chunked_exchange_both_directions(p, pattern, shape):
    """Plane-chunked exchange (TFFFT_FLAG_CHUNKED_EXCHANGE).  Forward: stage 1
    in plane chunks, each chunk's share of every band exchanged on the
    exchange stream while the next chunk computes.  Inverse: the bands are
    exchanged plane chunk after plane chunk and stage 1' (n1 columns + c2r
    rows) of a chunk runs as soon as it has landed, overlapping the next
    chunk's transfer.  Same spectra and real fields, bit for bit, as the
    unchunked plan, and the same wire bytes; (32, 1024, 16) puts the two-level
    warp-per-column kernel on the chunked n1 passes (plane offsets into the
    band tables and the landing buffer)."""
    x = oracle.uniform_field(shape, seed=7)
    grid = tf.GlobalGrid(*shape)
    slabs = tf.scatter_real(x, grid, p)

    def body(ep):
        out = []
        for algs in (("tma_columns",), ("chunked_exchange", "tma_columns")):
            fp = tf.plan(grid, ep, comm_pattern=pattern, algorithms=algs)
            assert ("chunked_exchange" in fp.algorithms) == ("chunked_exchange" in algs)
            spec = tf.forward(fp, slabs[ep.rank]).data.cpu().numpy().copy()
            wire_f = fp.counters.bytes_wire
            back = tf.inverse(fp, tf.forward(fp, slabs[ep.rank])).data.cpu().numpy().copy()
            wire = fp.counters.bytes_wire
            fp.close()
            out.append((spec, back, wire_f, wire))
        return out

    res = tf.run_spmd(p, body)
    ref = oracle.forward_all(x, p)
    n0p, n1p, n2c = shape[0] // p, shape[1] // p, shape[2] // 2 + 1
    band_bytes = (p - 1) * n0p * n1p * n2c * 16
    for q in range(p):
        plain, chunked = res[q]
        assert rel(chunked[0], ref[q]) <= 1e-12
        assert np.array_equal(chunked[0], plain[0]) and np.array_equal(chunked[1], plain[1])
        assert chunked[2] == band_bytes and chunked[3] == 3 * band_bytes  # forward, forward, inverse
        assert plain[3] == 3 * band_bytes
    back = np.concatenate([r[1][1] for r in res]).reshape(shape)
    assert rel(back, x) <= 1e-12


def test_deferred_consistency_mode():
    """check_consistency="deferred": every inverse folds the same Hermitian test
    on the device (no host sync per call); collect_consistency reports the
    calls checked and raises ConsistencyError for a bad spectrum in any of them."""
    shape = (16, 16, 16)
    grid = tf.GlobalGrid(*shape)
    ep = tf.make_communicators(1)[0]
    fp = tf.plan(grid, ep, check_consistency="deferred")
    slab = tf.scatter_real(oracle.uniform_field(shape, 4), grid, 1)[0]
    for _ in range(3):
        tf.inverse(fp, tf.forward(fp, slab))
    assert fp.collect_consistency() == 3
    assert 0.0 <= fp.last_imag_residue < 1e-9
    spec = tf.forward(fp, slab)
    spec.data.view(16, 16, 9)[5, 2, 8] += 1j  # one Nyquist bin becomes non-real
    tf.inverse(fp, spec)  # no exception at the call
    tf.inverse(fp, tf.forward(fp, slab))
    with pytest.raises(tf.ConsistencyError, match=r"in 2 inverse call\(s\)"):
        fp.collect_consistency()
    tf.inverse(fp, tf.forward(fp, slab))  # the accumulator was reset by the collect
    assert fp.collect_consistency() == 1
    fp.set_check_consistency(True)
    spec = tf.forward(fp, slab)
    spec.data.view(16, 16, 9)[5, 2, 8] += 1j
    with pytest.raises(tf.ConsistencyError):
        tf.inverse(fp, spec)
    fp.close()


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_nccl_calls_one_rank_loopback(dtype):
    """The exchange's NCCL calls through the dlopen'ed function table, as far as
    a one-GPU box can execute them (NCCL refuses two ranks on one device): a
    one-rank communicator, a grouped ncclSend / ncclRecv to self of one
    1024^3 p = 8 band chunk's worth of elements, ncclAlltoAll when the loaded
    NCCL has it, the one-int ncclAllReduce of the peer-store barrier and the
    async-error poll; the received payload must equal the sent one
    (tffft_nccl_loopback; exchange.py:263-290 over transport.py:359-419)."""
    count = 2 * 128 * 513 * 16  # real words of 16 planes of a 1024^3 p = 8 band
    try:
        ran_alltoall = tf.nccl_loopback(0, count, dtype)
    except tf.TransportError as e:
        if "NCCL unavailable" in str(e):
            pytest.skip(str(e))
        raise
    assert ran_alltoall in (True, False)
