"""GPU parity: libtffft forward/inverse against the CPU oracle (bit-pinned to
the reference) on seeded inputs.  Tolerances (BASELINE.json north_star):
relative L2 <= 1e-12 for float64, <= 1e-5 for float32, for the forward
spectrum and for the forward->inverse round trip."""

import glob
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1406_5597_b200 as tf

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TOL = {"float64": 1e-12, "float32": 1e-5}


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def run_pair(x, p, dtype="float64"):
    """forward + inverse on p ranks of the local fabric; returns per-rank flat
    spectral buffers (numpy), per-rank real outputs (numpy), residue."""
    shape = x.shape
    grid = tf.GlobalGrid(*shape)
    slabs = tf.scatter_real(x, grid, p, dtype=dtype)

    def body(ep):
        fp = tf.plan(grid, ep, tf.Strategy.STRIDED, dtype=dtype)
        spec = tf.forward(fp, slabs[ep.rank])
        f = spec.data.cpu().numpy().copy()
        back = tf.inverse(fp, spec)
        return f, back.data.cpu().numpy().copy(), fp.last_imag_residue

    res = tf.run_spmd(p, body)
    return [r[0] for r in res], [r[1] for r in res], max(r[2] for r in res)


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "ref_*.npz"))),
                         ids=lambda s: os.path.basename(s))
def test_golden_reference_vectors(path):
    """The GPU result against the reference's own outputs (fixtures)."""
    d = np.load(path)
    n0, n1, n2 = (int(v) for v in d["shape"])
    p = int(d["p"])
    gen = oracle.uniform_field if str(d["dist"]) == "uniform" else oracle.normal_field
    x = gen((n0, n1, n2), int(d["seed"]))
    fwd, inv, _ = run_pair(x, p)
    for q in range(p):
        assert rel(fwd[q], d["fwd"][q]) <= 1e-12
        assert rel(inv[q], d["inv"][q]) <= 1e-12


GRIDS = [
    ((2, 2, 2), 1), ((2, 2, 2), 2), ((4, 4, 4), 4), ((8, 8, 8), 1), ((16, 16, 16), 2),
    ((64, 64, 64), 1), ((32, 64, 128), 4), ((128, 16, 32), 8), ((16, 256, 64), 2),
    ((8, 8, 2048), 1), ((8, 2048, 4), 2), ((2048, 4, 8), 4), ((4096, 2, 2), 1), ((2, 4096, 4), 2),
    ((4, 4, 4096), 1), ((512, 8, 16), 8),
    # 1024-point transforms (two radix-32 passes) on every axis and path
    ((1024, 8, 16), 1), ((16, 1024, 8), 1), ((4, 8, 2048), 1), ((1024, 1024, 4), 2), ((1024, 16, 1024), 4),
]


@pytest.mark.parametrize("shape,p", GRIDS, ids=lambda v: str(v))
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_forward_inverse_vs_oracle(shape, p, dtype):
    x = oracle.uniform_field(shape, seed=sum(shape) + p)
    if dtype == "float32":
        x = x.astype(np.float32).astype(np.float64)  # identical values for both sides
    ref_flats = oracle.forward_all(x, p)
    fwd, inv, _ = run_pair(x, p, dtype)
    ref = oracle.gather_spectral(ref_flats, shape)
    got = oracle.gather_spectral([f.astype(np.complex128) for f in fwd], shape)
    assert rel(got, ref) <= TOL[dtype]
    # per-rank buffers are in the reference's STRIDED_INPLACE layout
    for q in range(p):
        assert rel(fwd[q], ref_flats[q]) <= TOL[dtype]
    back = np.concatenate([r.reshape(-1) for r in inv]).reshape(shape)
    assert rel(back, x) <= TOL[dtype]


def test_128_cubed_p2_layout_and_roundtrip():
    """BASELINE config 2: 128^3 float64 uniform, p=2: strided exchange layout + round trip."""
    shape = (128, 128, 128)
    x = oracle.uniform_field(shape, seed=2)
    ref_flats = oracle.forward_all(x, 2)
    fwd, inv, _ = run_pair(x, 2)
    for q in range(2):
        assert rel(fwd[q], ref_flats[q]) <= 1e-12
    assert rel(np.concatenate([r.reshape(-1) for r in inv]).reshape(shape), x) <= 1e-12


def test_64_cubed_p1_elementwise():
    """BASELINE config 1: 64^3 float64 uniform, p=1, elementwise vs the oracle."""
    shape = (64, 64, 64)
    x = oracle.uniform_field(shape, seed=1)
    ref = oracle.forward_all(x, 1)[0]
    fwd, inv, _ = run_pair(x, 1)
    assert np.max(np.abs(fwd[0] - ref)) <= 1e-10 * np.max(np.abs(ref))
    assert np.max(np.abs(inv[0].reshape(shape) - x)) <= 1e-13


def test_inverse_rejects_non_hermitian_spectrum():
    """kernels.py:225-238: imaginary DC/Nyquist bins raise ConsistencyError."""
    shape = (8, 8, 8)
    grid = tf.GlobalGrid(*shape)
    ep = tf.make_communicators(1)[0]
    fp = tf.plan(grid, ep)
    x = oracle.uniform_field(shape, 3)
    spec = tf.forward(fp, tf.scatter_real(x, grid, 1)[0])
    v = spec.data.view(8, 8, 5)
    v[1, 2, 0] += 1j  # DC bin of one row becomes non-real
    with pytest.raises(tf.ConsistencyError):
        tf.inverse(fp, spec)


def test_contract_errors():
    grid = tf.GlobalGrid(8, 8, 8)
    ep = tf.make_communicators(1)[0]
    fp = tf.plan(grid, ep)
    other = tf.scatter_real(np.zeros((8, 8, 8)), grid, 1, dtype="float32")[0]
    with pytest.raises(tf.ContractError):
        tf.forward(fp, other)
    spec = tf.SpectralSlab(fp.spectral_layout, tf.SpectralTag.CONTIGUOUS_FLIPPED, fp.work1)
    with pytest.raises(tf.ContractError):
        tf.inverse(fp, spec)


def test_counters_and_timers():
    shape = (16, 16, 16)
    x = oracle.uniform_field(shape, 5)
    grid = tf.GlobalGrid(*shape)
    slabs = tf.scatter_real(x, grid, 4)

    def body(ep):
        fp = tf.plan(grid, ep)
        fp.enable_timing()
        fp.reset_instrumentation()
        tf.inverse(fp, tf.forward(fp, slabs[ep.rank]))
        return fp.counters.snapshot(), fp.timers_us, fp.launches

    res = tf.run_spmd(4, body)
    chunk = 16 // 4 * 16 // 4 * 9 * 16
    for snap, timers, launches in res:
        # STRIDED: no pack / unpack pass, wire = off-rank bytes of two exchanges (transport.py:343-344)
        assert snap == (0, 2 * 3 * chunk, 0)
        assert set(timers) == {"stage1_us", "exchange_us", "stage3_us"}
        assert all(v >= 0 for v in timers.values())
        assert launches >= 6


ALG_CASES = [
    # fused stage 1 needs n1 == n2 in [512, 4096]; the four-step needs n0 in [512, 4096]
    ((4, 512, 512), 1, ("fused_stage1",)),
    ((8, 512, 512), 2, ("fused_stage1",)),
    ((512, 4, 8), 1, ("fourstep_stage3",)),
    ((512, 8, 16), 2, ("fourstep_stage3",)),
    ((1024, 4, 4), 4, ("fourstep_stage3",)),
    ((2048, 2, 4), 2, ("fourstep_stage3",)),
    ((4096, 2, 2), 1, ("fourstep_stage3",)),
    ((1024, 8, 8), 1, ("fourstep_stage3",)),      # TMA-fed four-step (p = 1)
    ((1024, 16, 64), 1, ("fourstep_stage3",)),
    ((8, 1024, 1024), 2, ("fused_stage1",)),
    ((2, 1024, 1024), 1, ("fused_stage1",)),
]


@pytest.mark.parametrize("shape,p,algs", ALG_CASES, ids=lambda v: str(v))
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_optional_schedules_vs_oracle(shape, p, algs, dtype):
    """The opt-in kernel schedules (fused persistent stage 1, L2-resident
    four-step stage 3) against the oracle, forward and round trip."""
    x = oracle.uniform_field(shape, seed=7 + p)
    if dtype == "float32":
        x = x.astype(np.float32).astype(np.float64)
    grid = tf.GlobalGrid(*shape)
    slabs = tf.scatter_real(x, grid, p, dtype=dtype)

    def body(ep):
        fp = tf.plan(grid, ep, tf.Strategy.STRIDED, dtype=dtype, algorithms=algs)
        # the optional schedules are single-rank kernels; p > 1 keeps the default ones
        assert set(fp.algorithms) == (set(algs) if p == 1 else set())
        spec = tf.forward(fp, slabs[ep.rank])
        f = spec.data.cpu().numpy().copy()
        back = tf.inverse(fp, spec)
        return f, back.data.cpu().numpy().copy()

    res = tf.run_spmd(p, body)
    ref = oracle.forward_all(x, p)
    for q in range(p):
        assert rel(res[q][0], ref[q]) <= TOL[dtype]
    back = np.concatenate([r[1].reshape(-1) for r in res]).reshape(shape)
    assert rel(back, x) <= TOL[dtype]


@pytest.mark.parametrize("algs", [(), ("fused_stage1", "fourstep_stage3")], ids=["default", "fused+fourstep"])
def test_512_cubed_normal_vs_torch_fft(algs):
    """BASELINE config 3 (512^3 float64 standard normal, p=1) at full size:
    forward against torch.fft.rfftn (test-only reference) and round trip."""
    import torch
    n = 512
    grid = tf.GlobalGrid(n, n, n)
    ep = tf.make_communicators(1)[0]
    fp = tf.plan(grid, ep, algorithms=algs)
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(n * n * n, dtype=torch.float64, device="cuda", generator=g)
    spec = tf.forward(fp, tf.RealSlab(fp.real_layout, x))
    ref = torch.fft.rfftn(x.view(n, n, n))
    err = (torch.linalg.norm(spec.data.view(n, n, n // 2 + 1) - ref) / torch.linalg.norm(ref)).item()
    assert err <= 1e-12
    back = tf.inverse(fp, spec)
    rt = (torch.linalg.norm(back.data - x) / torch.linalg.norm(x)).item()
    assert rt <= 1e-12


@pytest.mark.parametrize("shape,p", [((32, 32, 32), 2), ((16, 32, 8), 4), ((64, 64, 64), 1)])
def test_turbulence_batched_inverse_then_forward(shape, p):
    """BASELINE config 5 at small size: 3 velocity components built in Fourier
    space (white-noise phases x k^-5/3 radial amplitude, shell 1 <= |k| <= n/3),
    batched inverse c2r then forward r2c.  Spectra, real fields and the round
    trip are checked against the oracle (which also runs the reference's
    Hermitian consistency checks)."""
    grid = tf.GlobalGrid(*shape)
    kmax = shape[0] / 3
    noises = [oracle.normal_field(shape, 100 + c) for c in range(3)]
    amp = oracle.turbulence_amplitude(shape, 1.0, kmax)
    ref_specs = [oracle.gather_spectral(oracle.forward_all(w, p), shape) * amp for w in noises]
    n_slabs = [tf.scatter_real(w, grid, p) for w in noises]

    def body(ep):
        fp = tf.plan(grid, ep)
        specs = []
        for c in range(3):
            buf = torch.empty_like(fp.work1)
            specs.append(tf.turbulence_spectrum(fp, n_slabs[c][ep.rank], 1.0, kmax, out=buf))
        g_specs = [s.data.cpu().numpy().copy() for s in specs]
        reals = tf.inverse_batch(fp, specs, [torch.empty_like(fp.real_out) for _ in range(3)])
        r_np = [r.data.cpu().numpy().copy() for r in reals]
        back = tf.forward_batch(fp, reals, [torch.empty_like(fp.work1) for _ in range(3)])
        return g_specs, r_np, [b.data.cpu().numpy().copy() for b in back]

    res = tf.run_spmd(p, body)
    for c in range(3):
        got = oracle.gather_spectral([res[q][0][c] for q in range(p)], shape)
        assert rel(got, ref_specs[c]) <= 1e-12
        ref_real, _ = oracle.inverse_all(oracle.scatter_spectral(ref_specs[c], p), shape)
        for q in range(p):
            assert rel(res[q][1][c], ref_real[q].reshape(-1)) <= 1e-12
        back = oracle.gather_spectral([res[q][2][c] for q in range(p)], shape)
        assert rel(back, ref_specs[c]) <= 1e-12


def test_host_pair_stream_matches_device_path():
    """The host-buffer streaming API (bench e2e) returns the same round trip
    as the device calls, for several steps in flight."""
    shape = (64, 64, 32)
    grid = tf.GlobalGrid(*shape)
    ep = tf.make_communicators(1)[0]
    fp = tf.plan(grid, ep)
    xs = [oracle.uniform_field(shape, 40 + i) for i in range(5)]
    h_in = [torch.from_numpy(x.reshape(-1).copy()).pin_memory() for x in xs]
    h_out = [torch.empty_like(h).pin_memory() for h in h_in]
    tf.HostPairStream(fp).run(h_in, h_out)
    for x, h in zip(xs, h_out):
        assert rel(h.numpy().reshape(shape), x) <= 1e-12


@pytest.mark.parametrize("shape,p", [((8, 8, 8), 1), ((16, 16, 16), 2), ((32, 16, 8), 4), ((16, 8, 32), 8),
                                     ((128, 128, 128), 2), ((64, 64, 64), 1)], ids=lambda v: str(v))
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_transpose_strategy_equivalence(shape, p, dtype):
    """Strategy.TRANSPOSE (pack -> exchange -> unpack, CONTIGUOUS_FLIPPED) gives
    the same logical spectrum as STRIDED bit for bit (cli.py:192-198 'strategy
    equivalence'), round-trips, and counts the reference's copy bytes:
    packed = wire = unpacked = off-rank bytes, vs STRIDED's (0, wire, 0)."""
    x = oracle.uniform_field(shape, seed=13 + p)
    if dtype == "float32":
        x = x.astype(np.float32).astype(np.float64)
    grid = tf.GlobalGrid(*shape)
    slabs = tf.scatter_real(x, grid, p, dtype=dtype)

    def body(ep):
        out = {}
        for strat in (tf.Strategy.STRIDED, tf.Strategy.TRANSPOSE):
            fp = tf.plan(grid, ep, strat, dtype=dtype)
            fp.reset_instrumentation()
            spec = tf.forward(fp, slabs[ep.rank])
            logical = spec.as_logical().cpu().numpy().copy()
            back = tf.inverse(fp, spec)
            out[strat] = (logical, back.data.cpu().numpy().copy(), fp.counters.snapshot(), spec.tag)
            fp.close()
        return out

    res = tf.run_spmd(p, body)
    n0p, n1p, n2c = shape[0] // p, shape[1] // p, shape[2] // 2 + 1
    esz = 16 if dtype == "float64" else 8
    off = (p - 1) * n0p * n1p * n2c * esz
    for q in range(p):
        s, t = res[q][tf.Strategy.STRIDED], res[q][tf.Strategy.TRANSPOSE]
        assert t[3] is tf.SpectralTag.CONTIGUOUS_FLIPPED and s[3] is tf.SpectralTag.STRIDED_INPLACE
        assert np.array_equal(s[0], t[0])                    # bitwise strategy equivalence
        assert rel(t[1].reshape(-1), x[q * n0p:(q + 1) * n0p].reshape(-1)) <= TOL[dtype]
        assert s[2] == (0, 2 * off, 0)
        assert t[2] == (2 * off, 2 * off, 2 * off)


@pytest.mark.parametrize("shape,p", [((16, 16, 16), 2), ((32, 16, 8), 4), ((16, 8, 32), 8), ((128, 128, 128), 2)],
                         ids=lambda v: str(v))
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_peer_store_exchange(shape, p, dtype):
    """Fused exchange: the stage-1 / stage-3' epilogues store
    peer bands straight into the peers' landing buffers; the exchange is a
    barrier.  Same spectra (bitwise) and round trip as the staged exchange,
    over repeated calls (the landing buffers are rewritten each time)."""
    x = oracle.uniform_field(shape, seed=21 + p)
    if dtype == "float32":
        x = x.astype(np.float32).astype(np.float64)
    grid = tf.GlobalGrid(*shape)
    slabs = tf.scatter_real(x, grid, p, dtype=dtype)

    def body(ep):
        ref = tf.plan(grid, ep, dtype=dtype, algorithms=())
        fp = tf.plan(grid, ep, dtype=dtype, algorithms=("peer_stores",))
        assert fp.algorithms == ("peer_stores",)
        want = tf.forward(ref, slabs[ep.rank]).data.cpu().numpy().copy()
        got, backs = [], []
        for _ in range(3):
            spec = tf.forward(fp, slabs[ep.rank])
            got.append(spec.data.cpu().numpy().copy())
            backs.append(tf.inverse(fp, spec).data.cpu().numpy().copy())
        return want, got, backs

    res = tf.run_spmd(p, body)
    n0p = shape[0] // p
    for q in range(p):
        want, got, backs = res[q]
        for g, b in zip(got, backs):
            assert np.array_equal(g, want)
            assert rel(b, x[q * n0p:(q + 1) * n0p].reshape(-1)) <= TOL[dtype]


@pytest.mark.parametrize("shape,p", [((8, 8, 8), 1), ((16, 16, 16), 2), ((32, 16, 8), 4), ((16, 8, 32), 8)],
                         ids=lambda v: str(v))
@pytest.mark.parametrize("strategy", ["strided", "transpose"])
def test_collective_pattern_matches_pairwise(shape, p, strategy):
    """CommPattern.COLLECTIVE (transport.py:395-419) delivers
    the same spectra bit for bit as PAIRWISE, matches the oracle, round-trips,
    and counts the same wire bytes."""
    x = oracle.uniform_field(shape, seed=31 + p)
    grid = tf.GlobalGrid(*shape)
    slabs = tf.scatter_real(x, grid, p)
    strat = tf.Strategy(strategy)

    def body(ep):
        out = {}
        for pat in (tf.CommPattern.PAIRWISE, tf.CommPattern.COLLECTIVE):
            fp = tf.plan(grid, ep, strat, pat)
            assert fp.comm_pattern is pat
            fp.reset_instrumentation()
            spec = tf.forward(fp, slabs[ep.rank])
            logical = spec.as_logical().cpu().numpy().copy()
            back = tf.inverse(fp, spec).data.cpu().numpy().copy()
            out[pat] = (logical, back, fp.counters.snapshot())
            fp.close()
        return out

    res = tf.run_spmd(p, body)
    n0p, n1p = shape[0] // p, shape[1] // p
    want = np.fft.rfftn(x)
    for q in range(p):
        a, b = res[q][tf.CommPattern.PAIRWISE], res[q][tf.CommPattern.COLLECTIVE]
        assert np.array_equal(a[0], b[0])
        assert a[2] == b[2]
        assert rel(b[0].reshape(-1), want[:, q * n1p:(q + 1) * n1p].transpose(1, 0, 2).reshape(-1)) <= 1e-12
        assert rel(b[1], x[q * n0p:(q + 1) * n0p].reshape(-1)) <= TOL["float64"]


TMA_CASES = [((512, 8, 8), 1), ((8, 1024, 16), 1), ((1024, 1024, 4), 1), ((512, 512, 8), 1), ((64, 512, 32), 2),
             ((1024, 64, 16), 2), ((512, 512, 8), 4), ((1024, 32, 64), 8), ((32, 1024, 16), 4),
             ((1024, 16, 8), 16)]


@pytest.mark.parametrize("shape,p", TMA_CASES, ids=lambda v: str(v))
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_tma_column_kernel_bitwise(shape, p, dtype):
    """TMA-fed column passes (col_tma.cuh, lengths 512 / 1024): the same
    Stockham arithmetic as the cp.async kernel, so spectra and inverse outputs
    are bitwise identical to the cp.async kernels, and within tolerance of the
    oracle.  Covers partial tiles (columns not a multiple of the box width),
    float32 stage 1b (row stride not 16-byte aligned: falls back), and p > 1:
    the two-level variant (4D landing loads, block-table stores) at
    p = 2 .. 16, including blocks shorter than a 256-row box."""
    x = oracle.uniform_field(shape, seed=31)
    if dtype == "float32":
        x = x.astype(np.float32).astype(np.float64)
    grid = tf.GlobalGrid(*shape)
    slabs = tf.scatter_real(x, grid, p, dtype=dtype)

    def body(ep):
        ref = tf.plan(grid, ep, dtype=dtype, algorithms=())
        fp = tf.plan(grid, ep, dtype=dtype, algorithms=("tma_columns",))
        assert fp.algorithms == ("tma_columns",)
        want = tf.forward(ref, slabs[ep.rank]).data.clone()
        want_back = tf.inverse(ref, tf.SpectralSlab(ref.spectral_layout, tf.SpectralTag.STRIDED_INPLACE,
                                                      want.clone())).data.clone()
        got = tf.forward(fp, slabs[ep.rank]).data.clone()
        back = tf.inverse(fp, tf.SpectralSlab(fp.spectral_layout, tf.SpectralTag.STRIDED_INPLACE,
                                              got.clone())).data.clone()
        return (want.cpu().numpy(), want_back.cpu().numpy(), got.cpu().numpy(), back.cpu().numpy())

    res = tf.run_spmd(p, body)
    ref = oracle.forward_all(x, p)
    n0p = shape[0] // p
    for q in range(p):
        want, want_back, got, back = res[q]
        assert np.array_equal(got, want)
        assert np.array_equal(back, want_back)
        assert rel(got, ref[q]) <= TOL[dtype]
        assert rel(back, x[q * n0p:(q + 1) * n0p].reshape(-1)) <= TOL[dtype]


WPC_CASES = [((1024, 16, 8), 1), ((8, 1024, 16), 1), ((1024, 1024, 4), 1), ((16, 1024, 64), 1),
             ((32, 1024, 16), 2), ((32, 1024, 16), 4), ((64, 1024, 16), 8), ((16, 1024, 8), 16),
             ((1024, 64, 16), 2), ((1024, 32, 16), 8),
             ((512, 16, 8), 1), ((8, 512, 16), 1), ((512, 512, 8), 1), ((32, 512, 16), 4), ((512, 64, 16), 2),
             ((512, 32, 16), 8), ((16, 512, 8), 16),
             # one spectral row per rank (n1p = 1): an odd number of columns per rank, which the float32
             # TMA stores must not take (whole 16-byte chunks)
             ((1024, 2, 4), 2), ((512, 4, 8), 4)]


@pytest.mark.parametrize("shape,p", WPC_CASES, ids=lambda v: str(v))
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_wpc_column_kernel_bitwise(shape, p, dtype, monkeypatch):
    """Warp-per-column kernel (col_wpc.cuh, 1024-point columns, and 512-point
    columns two per warp with two sub-boxes side by side): one warp owns a
    column, operands from the swizzled TMA landing ring, outputs through TMA
    stores.  Same engine and twiddles as col_tma_kernel, so with it on every
    1024-point pass (TFFFT_WPC=1), on the stage-1b passes only (the default,
    2) or off (0) the spectra and inverse outputs are bitwise identical, and
    within tolerance of the oracle.  Covers partial tiles (n2c = 5, 9, 33
    columns per group), more CTAs than tiles, the float32 stage-1b rows that
    miss 16-byte alignment (fall back to col_tma_kernel), and p > 1: forward
    stage 1b storing every band through its own tensor map (band redirects),
    inverse stage 1b' loading the landing bands through the 4D map, with
    blocks of 512 down to 64 rows."""
    x = oracle.uniform_field(shape, seed=37)
    if dtype == "float32":
        x = x.astype(np.float32).astype(np.float64)
    grid = tf.GlobalGrid(*shape)
    slabs = tf.scatter_real(x, grid, p, dtype=dtype)

    def body(ep):
        fp = tf.plan(grid, ep, dtype=dtype)
        for _ in range(2):  # twice: the ticket counter and the mbarrier phases start over per launch
            spec = tf.forward(fp, slabs[ep.rank]).data.clone()
            back = tf.inverse(fp, tf.SpectralSlab(fp.spectral_layout, tf.SpectralTag.STRIDED_INPLACE,
                                                  spec.clone())).data.clone()
        res = (spec.cpu().numpy(), back.cpu().numpy())
        fp.close()
        return res

    out = {}
    for mode in ("0", "1", "2"):
        monkeypatch.setenv("TFFFT_WPC", mode)
        out[mode] = tf.run_spmd(p, body)
    ref = oracle.forward_all(x, p)
    n0p = shape[0] // p
    for q in range(p):
        for mode in ("1", "2"):
            assert np.array_equal(out[mode][q][0], out["0"][q][0])
            assert np.array_equal(out[mode][q][1], out["0"][q][1])
        assert rel(out["2"][q][0], ref[q]) <= TOL[dtype]
        assert rel(out["2"][q][1], x[q * n0p:(q + 1) * n0p].reshape(-1)) <= TOL[dtype]


WPC2_CASES = [((2048, 16, 8), 1), ((8, 2048, 16), 1), ((2048, 2048, 4), 1), ((16, 2048, 64), 1),
              ((2048, 32, 16), 2), ((32, 2048, 16), 4), ((2048, 2048, 2), 8), ((64, 2048, 8), 16),
              ((2048, 64, 4), 64), ((2048, 2, 4), 2)]


@pytest.mark.parametrize("shape,p", WPC2_CASES, ids=lambda v: str(v))
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_wpc2_2048_point_columns_vs_oracle(shape, p, dtype, monkeypatch):
    """2048-point columns as 2 x 1024 on the warp-per-column kernel with the
    even half parked in tensor memory (col_wpc2.cuh): stage 1b / 1b' (n1 =
    2048) and stage 3 / 3' (n0 = 2048), p = 1 and the two-level variants
    (row-parity 5D landing loads, one store map per destination block) down
    to blocks of 32 rows (p = 64: 16 half rows per sub-box).  Against the
    oracle, and against col_fft_kernel (TFFFT_WPC=0) within the same
    tolerance (a different factorisation: not bitwise)."""
    x = oracle.uniform_field(shape, seed=41)
    if dtype == "float32":
        x = x.astype(np.float32).astype(np.float64)
    grid = tf.GlobalGrid(*shape)
    slabs = tf.scatter_real(x, grid, p, dtype=dtype)

    def body(ep):
        fp = tf.plan(grid, ep, dtype=dtype)
        for _ in range(2):
            spec = tf.forward(fp, slabs[ep.rank]).data.clone()
            back = tf.inverse(fp, tf.SpectralSlab(fp.spectral_layout, tf.SpectralTag.STRIDED_INPLACE,
                                                  spec.clone())).data.clone()
        res = (spec.cpu().numpy(), back.cpu().numpy())
        fp.close()
        return res

    out = {}
    for mode in ("0", "2"):
        monkeypatch.setenv("TFFFT_WPC", mode)
        out[mode] = tf.run_spmd(p, body)
    ref = oracle.forward_all(x, p)
    n0p = shape[0] // p
    for q in range(p):
        assert rel(out["2"][q][0], ref[q]) <= TOL[dtype]
        assert rel(out["2"][q][1], x[q * n0p:(q + 1) * n0p].reshape(-1)) <= TOL[dtype]
        assert rel(out["2"][q][0], out["0"][q][0]) <= TOL[dtype]


@pytest.mark.parametrize("p", [1, 2, 4])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_constant_and_delta_known_answers(p, dtype):
    """SPEC.md known answers on the GPU path: a constant field has only the DC
    bin (n0 n1 n2 c) and a delta at the origin has every bin equal to 1; the
    inverse returns the field."""
    shape = (16, 8, 32)
    grid = tf.GlobalGrid(*shape)
    n = shape[0] * shape[1] * shape[2]
    for kind in ("constant", "delta"):
        x = np.full(shape, 0.75) if kind == "constant" else np.zeros(shape)
        if kind == "delta":
            x[0, 0, 0] = 1.0
        slabs = tf.scatter_real(x, grid, p, dtype=dtype)

        def body(ep):
            fp = tf.plan(grid, ep, dtype=dtype)
            spec = tf.forward(fp, slabs[ep.rank])
            s = tf.SpectralSlab(fp.spectral_layout, tf.SpectralTag.STRIDED_INPLACE, spec.data.clone())
            back = tf.inverse(fp, spec)
            return s, tf.RealSlab(fp.real_layout, back.data.clone())

        res = tf.run_spmd(p, body)
        g = tf.gather_spectral([r[0] for r in res])
        want = np.zeros(g.shape, dtype=np.complex128)
        if kind == "constant":
            want[0, 0, 0] = 0.75 * n
        else:
            want[...] = 1.0
        tol = TOL[dtype] * max(1.0, np.abs(want).max())
        assert np.max(np.abs(g - want)) <= tol * 10
        back = tf.gather_real([r[1] for r in res])
        assert np.max(np.abs(back - x)) <= TOL[dtype] * 10
