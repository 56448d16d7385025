"""Host-buffer streaming of forward+inverse pairs (the end-to-end path).

A user whose fields live in host memory calls ``HostPairStream(fp).run(...)``:
every step copies that step's real slab host->device, runs the forward r2c and
inverse c2r through libtffft and copies the result device->host.  Copies run
on their own CUDA streams and are double-buffered, so step i+1's upload and
step i's download (PCIe is full duplex) overlap the transforms of the
neighbouring steps instead of serialising with them.  With a plan made with
``check_consistency="deferred"`` no step waits for the host: every inverse's
Hermitian check is folded on the device and collected once at the end.
"""

from __future__ import annotations

import torch

from .dfft import FftPlan, forward, forward_many, inverse, inverse_many
from .layout import RealSlab

__all__ = ["HostPairStream"]


class HostPairStream:
    def __init__(self, fp: FftPlan, depth: int = 2):
        self.fp = fp
        self.depth = depth
        dev = fp.device
        self.d_in = [torch.empty_like(fp.real_out) for _ in range(depth)]
        self.d_out = [torch.empty_like(fp.real_out) for _ in range(depth)]
        self.h2d = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        self.compute = torch.cuda.current_stream(dev)

    def run(self, host_in: list[torch.Tensor], host_out: list[torch.Tensor]) -> None:
        """Transform host_in[i] -> host_out[i] (pinned host tensors of the real
        slab size, times fp.batch for a batched plan) for every i; returns when
        all results are on the host."""
        fp, dev = self.fp, self.fp.device
        n, depth = len(host_in), self.depth
        in_ready = [torch.cuda.Event() for _ in range(n)]
        in_free = [torch.cuda.Event() for _ in range(n)]
        out_ready = [torch.cuda.Event() for _ in range(n)]
        out_free = [torch.cuda.Event() for _ in range(n)]

        def upload(i):
            b = i % depth
            with torch.cuda.stream(self.h2d):
                if i >= depth:
                    self.h2d.wait_event(in_free[i - depth])   # forward(i - depth) consumed the buffer
                self.d_in[b].copy_(host_in[i], non_blocking=True)
                in_ready[i].record(self.h2d)

        for i in range(min(depth, n)):
            upload(i)
        for i in range(n):
            b = i % depth
            with torch.cuda.stream(self.compute):
                self.compute.wait_event(in_ready[i])
                if i >= depth:
                    self.compute.wait_event(out_free[i - depth])  # download(i - depth) done
                if fp.batch > 1:  # a batched plan: every step carries fp.batch fields
                    spec = forward_many(fp, self.d_in[b])
                    in_free[i].record(self.compute)
                    inverse_many(fp, spec, out=self.d_out[b])
                else:
                    spec = forward(fp, RealSlab(fp.real_layout, self.d_in[b]))
                    in_free[i].record(self.compute)
                    inverse(fp, spec, out=self.d_out[b])
                out_ready[i].record(self.compute)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(out_ready[i])
                host_out[i].copy_(self.d_out[b], non_blocking=True)
                out_free[i].record(self.d2h)
            if i + depth < n:
                upload(i + depth)
        self.d2h.synchronize()
        torch.cuda.current_stream(dev).synchronize()
        if fp.check_consistency == "deferred":  # every step's inverse was checked on the device
            fp.collect_consistency()
