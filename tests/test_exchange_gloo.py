"""Multi-rank host path on CPU (gloo, world_size 2 and 4): each rank takes
the oracle's stage-1 output, splits it the way the GPU stage-1 epilogue does
(every band through band_dst: the self band to landing[rank] -- or, for the
NCCL all-to-all, to the self slot staging[rank] -- and peer bands to
staging[q][i][j][k]), executes libtffft's exchange schedule with
torch.distributed send/recv into the landing buffer, reads every block from the
landing buffer through the STRIDED_INPLACE addressing the way the GPU stage-3
kernel does, runs the oracle's stage 3 and must land bit-exactly on the
reference's forward output."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, shape, q, pattern="pairwise"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1406_5597_b200 as tf

        n0, n1, n2 = shape
        x = oracle.normal_field(shape, 11)
        n0p = n0 // world
        s1 = oracle.stage1_forward(x[rank * n0p:(rank + 1) * n0p])
        spec, staging = oracle.stage1_band_staging(s1, world, rank)
        n1p, n2c = n1 // world, n2 // 2 + 1
        self_band = s1[:, rank * n1p:(rank + 1) * n1p]
        landing = torch.zeros(staging.size, dtype=torch.complex128)
        if pattern == "collective":
            # TFFFT_COLLECTIVE: one all-to-all over the p-band staging / landing
            # buffers; the self band rides in the self slot staging[rank]
            staging[rank] = self_band
            stg = torch.from_numpy(staging.reshape(-1).copy())
            dist.all_to_all_single(torch.view_as_real(landing), torch.view_as_real(stg))
        else:
            stg = torch.from_numpy(staging.reshape(-1).copy())
            landing.view(world, -1)[rank] = torch.from_numpy(self_band.reshape(-1).copy())  # band_dst[rank]
            ops = tf.exchange_schedule(n0, n1, n2, world, rank)
            reqs = []
            for op in ops:  # libtffft posts all sends and receives of a rank in one group
                reqs.append(dist.isend(stg[op.send_offset:op.send_offset + op.count].clone(), op.peer))
            for op in ops:
                reqs.append(dist.irecv(landing[op.recv_offset:op.recv_offset + op.count], op.peer))
            for r in reqs:
                r.wait()
        # the stage-3 kernel's read addressing: block s of a column comes from
        # landing[s][i][j][k]; its output is written in place, STRIDED_INPLACE
        lnd = landing.numpy().reshape(world, n0p, n1p, n2c)
        out = np.ascontiguousarray(lnd.transpose(1, 0, 2, 3)).reshape(-1)
        oracle.stage3(out, n0, n1, n2, world, inverse=False)
        ref = oracle.forward_all(x, world)[rank]
        q.put((rank, bool(np.array_equal(out.view(np.float64), ref.view(np.float64)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("pattern", ["pairwise", "collective"])
@pytest.mark.parametrize("world,shape", [(2, (8, 8, 8)), (2, (16, 4, 32)), (4, (8, 16, 4))])
def test_exchange_schedule_over_gloo(world, shape, pattern):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, q, pattern)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(res[r] for r in range(world)), res


def _peer_store_worker(rank, world, port, shape, landings, q):
    """Fused exchange over NCCL (peer stores through CUDA IPC mappings), host
    protocol on CPU: every rank publishes a 64-byte handle of its landing
    buffer, tf.allgather_handles returns them in rank order, and the stage-1
    epilogue's destination for band q is `landing of rank q + rank * band`
    (tffft.cu build_band_dst).  Shared-memory tensors stand in for the mapped
    peer buffers, dist.barrier for the one-int ncclAllReduce barrier."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1406_5597_b200 as tf

        n0, n1, n2 = shape
        n0p, n1p, n2c = n0 // world, n1 // world, n2 // 2 + 1
        band = n0p * n1p * n2c
        # a handle: 64 bytes naming this rank's landing buffer (index + padding)
        handle = rank.to_bytes(4, "little") + bytes(60)
        allh = tf.allgather_handles(handle, rank, world)
        assert len(allh) == 64 * world
        peers = [int.from_bytes(allh[64 * r:64 * r + 4], "little") for r in range(world)]
        assert peers == list(range(world))
        for _ in range(2):  # two calls: the guard barrier orders reuse of the landing buffers
            dist.barrier()  # guard: every peer has consumed its landing buffer
            x = oracle.normal_field(shape, 13)
            s1 = oracle.stage1_forward(x[rank * n0p:(rank + 1) * n0p])
            spec, staging = oracle.stage1_band_staging(s1, world, rank)
            stg = staging.reshape(world, band)
            stg[rank] = s1[:, rank * n1p:(rank + 1) * n1p].reshape(-1)
            for qq in range(world):  # epilogue stores: band qq -> landing of rank qq, block `rank`
                dst = landings[peers[qq]].numpy().reshape(world, band)  # (qq == rank: our own landing)
                dst[rank] = stg[qq]
            dist.barrier()  # the exchange: every rank's stores are visible
            lnd = landings[rank].numpy().reshape(world, n0p, n1p, n2c)
            out = np.ascontiguousarray(lnd.transpose(1, 0, 2, 3)).reshape(-1)
            oracle.stage3(out, n0, n1, n2, world, inverse=False)
            ref = oracle.forward_all(x, world)[rank]
            ok = bool(np.array_equal(out.view(np.float64), ref.view(np.float64)))
            if not ok:
                break
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape", [(2, (8, 8, 8)), (4, (8, 16, 4))])
def test_peer_store_protocol_over_gloo(world, shape):
    n0, n1, n2 = shape
    band = (n0 // world) * (n1 // world) * (n2 // 2 + 1)
    landings = [torch.zeros(world * band, dtype=torch.complex128).share_memory_() for _ in range(world)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_store_worker, args=(r, world, port, shape, landings, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(res[r] for r in range(world)), res


def _ipc_host_worker(rank, world, port, q):
    """IPC communicator host path (tffft_comm_init_ipc) on CPU: the gloo
    group's barrier reaches the library through the ctypes callback
    (tffft_comm_barrier), and plan blobs all-gather in rank order."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1406_5597_b200 as tf
        from paper_1406_5597_b200 import _lib

        ep = tf.init_ipc_endpoint(device=0)
        ok = ep.kind == "ipc" and ep.rank == rank and ep.p == world
        for _ in range(3):
            _lib.check(_lib.lib().tffft_comm_barrier(ep.handle))
        blob = bytes([rank]) * 256
        got = ep.allgather_bytes(blob)
        ok = ok and got == b"".join(bytes([r]) * 256 for r in range(world))
        ep.close()
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ipc_comm_host_protocol_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_host_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(res[r] for r in range(world)), res
