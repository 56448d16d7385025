"""Benchmark: 3D r2c+c2r FFT pair (forward + inverse) on B200 through libtffft.

Default workload (BASELINE.json headline): 1024^3 float64, slab-decomposed
over the N GPUs of the job (strong scaling; p = N).  Prints ONE JSON line.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--grid 1024] [--dtype float64]
  python bench.py --impl reference ...   # CPU oracle port of the reference path

value  = GFLOP/s of the whole job, 2 * 2.5 N log2 N per pair, inputs resident in
         HBM, device-timed (CUDA events, barrier + synchronize both sides, max
         over ranks).  The inputs (8.6 GB/slab at p=1) are far larger than L2.
e2e    = the same metric through the public API with host buffers: pinned-host
         -> device copy of the real slab, forward, inverse, device -> host copy
         of the result, all inside the timed region.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "3D r2c+c2r FFT pair: ms & GFLOP/s at 1/2/4/8 B200, % of HBM/NVLink roofline"
HBM_FALLBACK = 6650.0   # GB/s, B200_PROFILING.md fallback
NVLINK_GBS = 770.0      # measured peer copy per direction (B200_PROFILING.md)


def pair_flops(n0, n1, n2):
    n = n0 * n1 * n2
    return 2 * 2.5 * n * math.log2(n)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


def algorithmic_bytes(n0, n1, n2, p, s_r):
    """HBM bytes per GPU per pair, NVLink bytes per GPU per pair,
    and the bytes of one stage-3 launch (read + write of the spectral slab)."""
    n, nc = n0 * n1 * n2, n0 * n1 * (n2 // 2 + 1)
    s_c = 2 * s_r
    hbm = 2 * (s_r * n + 3 * s_c * nc) / p
    nvl = 2 * s_c * nc * (p - 1) / (p * p)
    stage3 = 2 * s_c * nc / p
    return hbm, nvl, stage3


class ClockSampler:
    """SM clocks, power and clock-event (throttle) reasons sampled during the
    timed region: NVML in-process every 10 ms (the device matched by PCI bus
    id), else nvidia-smi every ~0.2 s."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, {reason names}, watts)
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            prop = torch.cuda.get_device_properties(device)  # integer PCI ids
            want = (prop.pci_domain_id, prop.pci_bus_id, prop.pci_device_id)
            self._h = None
            for i in range(nv.nvmlDeviceGetCount()):
                h = nv.nvmlDeviceGetHandleByIndex(i)
                pci = nv.nvmlDeviceGetPciInfo(h)
                if (pci.domain, pci.bus, pci.device) == want:
                    self._h = h
                    break
            if self._h is None:
                raise RuntimeError("no NVML device with the CUDA device's PCI id")
            self._bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                          "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                          "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                          "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            self._nvml = nv
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv, h = self._nvml, self._h
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        # instantaneous board power: nvmlDeviceGetPowerUsage is a 1 s average,
        # which lags a sub-second timed region that starts from idle
        watts = None
        try:
            fv = nv.nvmlDeviceGetFieldValues(h, [nv.NVML_FI_DEV_POWER_INSTANT])[0]
            if fv.nvmlReturn == 0:
                watts = fv.value.uiVal / 1000.0
        except Exception:
            pass
        if watts is None:
            watts = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
        return (float(sm), float(mx), {n for n, b in self._bits.items() if bits & b}, watts)

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        f = [x.strip() for x in out.split(",")]
        num = lambda x: float(x) if x.replace(".", "").isdigit() else None
        return (num(f[0]), num(f[1]), {n for n, v in zip(self.NAMES, f[2:6]) if "Active" in v and "Not" not in v},
                num(f[6]) if len(f) > 6 else None)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample_nvml() if self._nvml else self._sample_smi())
            except Exception:
                return
            self._stop.wait(0.01 if self._nvml else 0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return None
        sm = [s[0] for s in self.samples if s[0] is not None]
        mx = [s[1] for s in self.samples if s[1] is not None]
        w = [s[3] for s in self.samples if s[3] is not None]
        reasons = sorted(set().union(*[s[2] for s in self.samples]))
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_min_mhz": min(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w_median": statistics.median(w) if w else None,
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi"}


# ---------------------------------------------------------------------------
# CPU oracle (reference path port): bounded sample of the same workload
# ---------------------------------------------------------------------------

def cpu_sample(n0, n1, n2, planes=64, workers=None):
    """Time the oracle (restatement of the reference's STRIDED pipeline,
    bit-identical to it) on a bounded sample of the full-size p = 1 pair:
    stage 1 + 1' (r2c rows, n1 columns and back) on `planes` of the n0
    planes, and stage 3 + 3' on the same fraction of the n1*n2c STRIDED_INPLACE
    columns, gathered and scattered at their true two-level offsets
    (layout.py:189-219) in a full-size spectral buffer.  Returns the MEASURED
    throughput of the sample (its own flops / its own seconds), the measured
    seconds, the threads used and a description.  Nothing is extrapolated."""
    import numpy as np

    import oracle

    workers = workers or len(os.sched_getaffinity(0))
    n2c = n2 // 2 + 1
    rng = np.random.default_rng(0)
    slab = rng.uniform(-1.0, 1.0, size=(planes, n1, n2))
    ncols = max(1, (n1 * n2c * planes) // n0)
    # full-size STRIDED_INPLACE buffer (p = 1: element r of column c at r*n1*n2c + c);
    # np.zeros maps pages lazily, so only the sampled columns' rows are touched
    flat = np.zeros(n0 * n1 * n2c, dtype=np.complex128)
    row = np.arange(n0, dtype=np.int64) * (n1 * n2c)
    blk = max(1, -(-ncols // (4 * workers)))
    spans = [(a, min(a + blk, ncols)) for a in range(0, ncols, blk)]
    for a, b in spans:
        offs = np.arange(a, b, dtype=np.int64)[:, None] + row[None, :]
        flat[offs] = rng.standard_normal(offs.shape) + 1j * rng.standard_normal(offs.shape)
    t0 = time.perf_counter()
    spec = oracle.stage1_forward(slab, workers)
    oracle.stage1_inverse(spec, n2, workers)
    t1 = time.perf_counter()
    for inv in (False, True):
        def work(a, b, inv=inv):
            offs = np.arange(a, b, dtype=np.int64)[:, None] + row[None, :]
            cols = flat[offs]
            oracle.c2c_rows(cols, inv)
            flat[offs] = cols
        oracle.slabfft_oracle._run(work, spans, workers)
    t2 = time.perf_counter()
    # flops of the sample: the pair's 2 * 2.5 N log2 N split over the axes as the
    # passes that ran (stage 1+1': planes/n0 of the n1 and n2 axis work; stage
    # 3+3': ncols/(n1*n2c) of the n0 axis work)
    n = n0 * n1 * n2
    f_axis = lambda L: 2 * 2.5 * n * math.log2(L)
    flops = f_axis(n1 * n2) * planes / n0 + f_axis(n0) * ncols / (n1 * n2c)
    secs = t2 - t0
    sample = (f"oracle port (bit-identical to the reference), {workers} threads, measured on a sample of the "
              f"{n0}x{n1}x{n2} float64 p=1 pair: stage 1+1' on {planes}/{n0} planes ({t1 - t0:.2f} s) and "
              f"stage 3+3' on {ncols}/{n1 * n2c} columns at their STRIDED_INPLACE offsets ({t2 - t1:.2f} s); "
              f"value = the sample's flops / its measured seconds")
    return flops / secs / 1e9, secs, workers, sample


def full_pair_record():
    """The one full-size CPU pair measured on the GPU host (tools/cpu_full_pair.py), if committed."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_cpu_full_pair.json")) as f:
            return json.load(f)
    except Exception:
        return None


def stage3_kernel_name(n0: int, dt: str) -> str:
    """The kernel the library runs for the stage-3 column pass by default (csrc/tffft.cu columns_wpc /
    columns_tma): float64 1024-point columns keep col_tma_kernel; 512-point, float32 1024-point and
    2048-point columns run the warp-per-column kernels; other lengths col_fft_kernel."""
    if os.environ.get("TFFFT_TMA_COLS") == "0":
        return "col_fft_kernel"
    wpc = os.environ.get("TFFFT_WPC", "2")
    if n0 == 2048 and wpc != "0":
        return "col_wpc2_kernel"
    if n0 == 512 and wpc != "0":
        return "col_wpc_kernel"
    if n0 == 1024:
        return "col_wpc_kernel" if (wpc == "1" or (wpc == "2" and dt == "float32")) else "col_tma_kernel"
    return "col_tma_kernel" if n0 == 512 else "col_fft_kernel"


def cube_config(n0, n1, n2, dt, p):
    """The config object both arms print (identical keys and values)."""
    s_r = 8 if dt == "float64" else 4
    return {"workload": f"{n0}x{n1}x{n2} {dt} r2c+c2r pair, slab p={p}",
            "grid": [n0, n1, n2], "p": p, "parallelism": f"slab{p}",
            "l2": f"inputs larger than L2 ({n0 // p * n1 * n2 * s_r / 1e9:.2f} GB real slab per GPU)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n0 = n1 = n2 = args.grid
    # one step = one measured sample of the workload (cpu_sample); ms_per_step is
    # that measured time, so steps x ms_per_step is the real timed region
    vals = []
    for i in range(args.warmup + args.steps):
        gf, secs, cores, sample = cpu_sample(n0, n1, n2, planes=args.cpu_planes)
        if i >= args.warmup:
            vals.append((gf, secs))
    gf = statistics.median(v[0] for v in vals)
    ms = statistics.median(v[1] for v in vals) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": gf, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        # the GPU arm's config object, key for key; the CPU port computes the whole
        # pair, which is what the p slabs compute together
        "config": cube_config(n0, n1, n2, "float64", args.gpus),
        "cpu_baseline": {"value": gf, "unit": "GFLOP/s", "cores": cores, "kind": "port", "sample": sample,
                         "timed_steps_s": [round(v[1], 3) for v in vals]},
        "e2e": {"value": gf, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    full = full_pair_record()
    if full and full.get("grid") == [n0, n1, n2]:
        line["cpu_full_pair"] = full
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_1406_5597_b200 as tf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        ep = tf.init_nccl_endpoint(local)
    else:
        ep = tf.make_communicators(1, device=local)[0]
    p = world
    n0 = n1 = n2 = args.grid
    grid = tf.GlobalGrid(n0, n1, n2)
    dt = args.dtype
    s_r = 8 if dt == "float64" else 4
    # the reference's inverse checks the half spectrum on every call
    # (kernels.py:223-238): so does the timed pair (reduction + host check)
    ncomp = 3 if args.config == "turbulence" else 1
    # turbulence: one batched plan for the 3 components (one launch per stage
    # over all of them at p = 1; exchange/compute overlap across them at p > 1)
    fp = tf.plan(grid, ep, tf.Strategy.STRIDED, dtype=dt, check_consistency=True, batch=ncomp)
    rdt = tf.DTYPES[dt][1]
    n0p = n0 // p
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    x = torch.empty(ncomp * n0p * n1 * n2, dtype=rdt, device=dev)
    x.uniform_(-1.0, 1.0, generator=gen)
    slab = tf.RealSlab(fp.real_layout, x) if ncomp == 1 else None
    stream = torch.cuda.current_stream(dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    tol = 1e-12 if dt == "float64" else 1e-5
    if args.config == "turbulence":
        # BASELINE config 5: 3 velocity components defined in Fourier space
        # (white-noise phases x k^-5/3 on 1 <= |k| <= 340), batched inverse c2r
        # then forward r2c.  One step = the batched round trip of all components.
        noise = torch.empty_like(x)
        noise.normal_(generator=gen)
        specs = tf.turbulence_spectra(fp, noise, 1.0, 340.0 * n0 / 1024, out=torch.empty_like(fp.work1))
        del noise
        reals = torch.empty_like(fp.real_out)
        ref0 = specs.view(ncomp, -1)[0].clone()

        def step():
            tf.inverse_many(fp, specs, out=reals)
            tf.forward_many(fp, reals, out=specs)
    else:
        def step():
            tf.inverse(fp, tf.forward(fp, slab))

    # correctness guard on the timed configuration (reference cli.py:263-271 style)
    step()
    torch.cuda.synchronize(dev)
    if args.config == "turbulence":
        rt = (torch.linalg.norm(specs.view(ncomp, -1)[0] - ref0) / torch.linalg.norm(ref0)).item()
        del ref0
    else:
        rt = (torch.linalg.norm(fp.real_out.double() - x.double()) / torch.linalg.norm(x.double())).item()
    if not rt <= tol:
        raise SystemExit(f"round-trip check failed: rel L2 {rt:.3e} > {tol}")

    for _ in range(args.warmup):
        step()
    barrier()
    fp.enable_timing(True)
    fp.reset_instrumentation()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        while not e1.query():  # wait without holding the GIL, so the clock sampler keeps sampling
            time.sleep(0.002)
        barrier()
    ms = e0.elapsed_time(e1) / args.steps
    launches = fp.launches
    stages = fp.timers_us
    fp.enable_timing(False)
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # e2e through the public API with host buffers: HostPairStream copies each
    # step's real slab host->device, runs the pair and copies the result back;
    # uploads and downloads of neighbouring steps overlap (PCIe full duplex)
    if args.config == "turbulence":
        del specs, reals
    h_in = torch.empty(ncomp * n0p * n1 * n2, dtype=rdt, pin_memory=True)
    h_in.copy_(x)
    h_out = torch.empty_like(h_in, pin_memory=True)
    # K steps like the device-timed region (the pipeline's fill and drain -- one
    # upload before the first pair, one download after the last -- are inside the
    # timed region and amortise over the K steps); --e2e-steps caps it
    e2e_steps = max(1, min(args.steps, args.e2e_steps) if args.e2e_steps > 0 else args.steps)
    # every step's inverse still runs the Hermitian check, folded on the device
    # and collected once per run (no host synchronisation per step)
    fp.set_check_consistency("deferred")
    streamer = tf.HostPairStream(fp)
    streamer.run([h_in], [h_out])  # warm-up
    barrier()
    t0 = time.perf_counter()
    streamer.run([h_in] * e2e_steps, [h_out] * e2e_steps)
    barrier()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    del streamer
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    flops = pair_flops(n0, n1, n2) * ncomp
    value = flops / (ms * 1e-3) / 1e9
    hbm_peak, peak_kind = peaks()
    hbm, nvl, st3 = algorithmic_bytes(n0, n1, n2, p, s_r)
    hbm, nvl = hbm * ncomp, nvl * ncomp
    t_roof = max(hbm / (hbm_peak * 1e9), nvl / (NVLINK_GBS * 1e9) if p > 1 else 0.0) * 1e3
    # dominant kernel: the stage-3 strided column c2c (one launch per direction)
    st3_ms = stages["stage3_us"] / 1e3 / (2 * args.steps * ncomp)
    st1_ms = stages["stage1_us"] / 1e3 / (2 * args.steps * ncomp)
    ach = st3 / (st3_ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "stage3_traffic.json")
    try:
        with open(tpath) as f:
            tr = json.load(f)
        key = f"{n0}x{n1}x{n2}_{dt}_p{p}"
        traffic = tr.get(key)
    except Exception:
        pass

    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64" if dt == "float64" else "f32",
        "data": "synthetic: seeded uniform[-1,1) real field generated on device",
        "config": (cube_config(n0, n1, n2, dt, p) if ncomp == 1 else
                   dict(cube_config(n0, n1, n2, dt, p),
                        workload=(f"turbulence: 3 x {n0}x{n1}x{n2} {dt} components, batched inverse c2r then "
                                  f"forward r2c, slab p={p}"))),
        "details": {
            "pair_roofline_ms": t_roof, "pair_roofline_frac": t_roof / ms,
            "stage_ms_per_pair": {"stage1+1'": st1_ms * 2,
                                  "exchange": stages["exchange_us"] / 1e3 / (args.steps * ncomp),
                                  "stage3+3'": st3_ms * 2},
            "roundtrip_rel_l2": rt,
        },
        "roofline": {"bound": "hbm",
                     "kernel": stage3_kernel_name(n0, dt) + " (stage 3 strided n0 c2c)",
                     "achieved": ach, "peak": hbm_peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": ach / hbm_peak, "traffic": traffic,
                     "algorithmic_bytes_per_launch": st3},
        "e2e": {"value": pair_flops(n0, n1, n2) * ncomp / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s", "ms_per_step": e2e_ms, "steps": e2e_steps,
                "api": ("paper_1406_5597_b200.HostPairStream (pinned host slab in, host slab out per step; the "
                        "Hermitian check of every inverse folded on the device, collected per run)"),
                "h2d_bytes_per_step": h_in.numel() * h_in.element_size(),
                "d2h_bytes_per_step": h_out.numel() * h_out.element_size()},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu and args.config == "cube":
        gf, _, cores, sample = cpu_sample(n0, n1, n2, planes=args.cpu_planes)
        line["cpu_baseline"] = {"value": gf, "unit": "GFLOP/s", "cores": cores, "kind": "port", "sample": sample}
        full = full_pair_record()
        if full and full.get("grid") == [n0, n1, n2] and dt == "float64":
            line["cpu_full_pair"] = full
    if rank == 0:
        print(json.dumps(line))
    fp.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--grid", type=int, default=1024)
    ap.add_argument("--dtype", choices=["float64", "float32"], default="float64")
    ap.add_argument("--config", choices=["cube", "turbulence"], default="cube",
                    help="cube: seeded uniform field pair (headline); turbulence: BASELINE config 5")
    ap.add_argument("--e2e-steps", type=int, default=0,
                    help="host-buffer (e2e) steps; 0 = the same K as --steps")
    ap.add_argument("--cpu-planes", type=int, default=64)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args.gpus)
    return run_gpu(args)


def self_launch(n):
    """`python bench.py --gpus N` outside torchrun: re-run this command as N
    ranks (one process per GPU) under torch.distributed.run on 127.0.0.1;
    rank 0 prints the JSON line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


if __name__ == "__main__":
    sys.exit(main())
