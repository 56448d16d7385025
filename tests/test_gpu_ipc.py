"""The cross-process exchange on a real GPU: p PROCESSES, one rank each, all
on cuda:0, with the IPC communicator (tffft_comm_init_ipc).

Each process exports its plan's staging / landing buffers and events as CUDA
IPC handles, the blobs are all-gathered over a gloo group, and every process
maps its peers' -- the handle export / attach path the NCCL peer-store
exchange also uses.  The exchange then runs across process boundaries: IPC
events order each rank's pull of its peers' staging bands (or, with peer
stores, the producing stage's stores straight into the peers' landing
buffers).  No kernel waits on another rank's kernel (the only cross-rank
waits are stream-event dependencies and the gloo host barrier), so the ranks
may time-share one GPU (B200_PROFILING.md: spinning ranks on one GPU raised
Xid 109; this transport never spins).

Every rank's STRIDED_INPLACE buffer must equal the oracle's for that rank
(relative L2 <= 1e-12) and the round trip must recover the input.
"""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = [
    # (shape, pattern, algorithms, batch)
    ((32, 32, 16), "PAIRWISE", None, 1),
    ((32, 32, 16), "COLLECTIVE", None, 1),
    ((32, 32, 16), "PAIRWISE", ("peer_stores",), 1),
    ((64, 32, 8), "PAIRWISE", None, 3),
    ((64, 32, 8), "COLLECTIVE", ("peer_stores",), 3),
    ((16, 1024, 8), "PAIRWISE", None, 1),
    ((64, 32, 16), "PAIRWISE", ("chunked_exchange", "tma_columns"), 1),
    ((64, 32, 16), "COLLECTIVE", ("chunked_exchange",), 1),
    # warp-per-column kernels storing through tensor maps over IPC-mapped peer landing buffers
    ((32, 1024, 16), "PAIRWISE", ("peer_stores", "tma_columns"), 1),   # stage 1b forward (1024 points)
    ((2048, 16, 8), "PAIRWISE", ("peer_stores", "tma_columns"), 1),    # stage 3' (2 x 1024 through tensor memory)
    ((512, 16, 8), "COLLECTIVE", ("peer_stores", "tma_columns"), 2),   # 512 points, batched pipeline
]


def _rank_main(rank, world, port, errfile):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import oracle
    import paper_1406_5597_b200 as tf

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    ep = tf.init_ipc_endpoint(0)
    assert ep.kind == "ipc" and ep.p == world and ep.rank == rank
    msgs = []
    for shape, pattern, algs, batch in CASES:
        grid = tf.GlobalGrid(*shape)
        fields = [oracle.uniform_field(shape, seed=sum(shape) + c) for c in range(batch)]
        refs = [oracle.forward_all(x, world)[rank] for x in fields]
        fp = tf.plan(grid, ep, tf.Strategy.STRIDED, comm_pattern=tf.CommPattern[pattern], algorithms=algs,
                     batch=batch)
        real = torch.cat([tf.scatter_real(x, grid, world)[rank].data for x in fields])
        for rep in range(2):  # twice: buffer and event reuse across calls
            spec = tf.forward_many(fp, real) if batch > 1 else tf.forward(fp, tf.RealSlab(fp.real_layout, real)).data
            got = spec.view(batch, -1).cpu().numpy()
            back = (tf.inverse_many(fp, spec) if batch > 1 else
                    tf.inverse(fp, tf.SpectralSlab(fp.spectral_layout, tf.SpectralTag.STRIDED_INPLACE, spec)).data)
            bk = back.view(batch, -1).cpu().numpy()
            for c in range(batch):
                e = np.linalg.norm(got[c] - refs[c]) / np.linalg.norm(refs[c])
                xr = real.view(batch, -1)[c].cpu().numpy()
                r = np.linalg.norm(bk[c] - xr) / np.linalg.norm(xr)
                if not (e <= 1e-12 and r <= 1e-12):
                    msgs.append(f"rank {rank} {shape} {pattern} {algs} b{batch} rep{rep} field {c}: fwd {e:.2e} rt {r:.2e}")
        wire = fp.counters.bytes_wire
        expect = 2 * 2 * batch * (world - 1) * (shape[0] // world) * (shape[1] // world) * (shape[2] // 2 + 1) * 16
        if wire != expect:
            msgs.append(f"rank {rank} {shape} {pattern}: wire bytes {wire} != {expect}")
        ep.barrier()  # no peer still references this plan's buffers or events
        fp.close()
    ep.barrier()
    ep.close()
    dist.destroy_process_group()
    if msgs:
        with open(errfile, "a") as f:
            f.write("\n".join(msgs) + "\n")


@pytest.mark.parametrize("world", [2, 4])
def test_ipc_exchange_across_processes(world, tmp_path):
    import torch.multiprocessing as mp

    errfile = str(tmp_path / "errors.txt")
    mp.spawn(_rank_main, args=(world, _free_port(), errfile), nprocs=world, join=True)
    if os.path.exists(errfile):
        pytest.fail(open(errfile).read())
