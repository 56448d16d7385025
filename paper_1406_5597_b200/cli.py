"""Command line tool of the B200 path, mirroring the reference CLI
(reference pkg/src/slabfft/cli.py:399-456):

  verify   oracle-equivalence and round-trip suites over a grid x procs
           cross product (cli.py:159-202); the brute-force DFT is a direct
           triple sum evaluated with torch on the device (oracle.py:30-45)
  bench    forward+inverse pairs, per-stage times and copy counters as CSV
           with the reference's header (cli.py:32-47, 319-339)
  compare  the paper's A/B: STRIDED (transpose-free) against TRANSPOSE on
           identical inputs, median times, copy-byte ratio and a bitwise
           strategy-equivalence check (cli.py:342-383)

Exit codes (cli.py:440-456): 0 all checks passed, 1 a check failed,
2 usage or configuration error.  Ranks are host threads over the in-process
fabric on one GPU (``run_spmd``), as in the reference's THREADED mode.
"""

from __future__ import annotations

import argparse
import csv
import math
import statistics
import sys

import torch

from .dfft import forward, gather_real, gather_spectral, inverse, plan, scatter_real
from .errors import ConfigurationError, SlabFftError
from .exchange import Strategy
from .layout import GlobalGrid, RealSlab, SpectralSlab, validate
from .transport import CommPattern, run_spmd

MAX_VERIFY_SIZE = 32  # cli.py:30
ROUNDTRIP_RTOL = 1e-12  # cli.py:49
ORACLE_ATOL = 1e-10  # cli.py:50
CSV_COLUMNS = [
    "grid_n0", "grid_n1", "grid_n2", "p", "strategy", "comm_pattern", "iter", "t_total_us", "t_stage1_us",
    "t_exchange_us", "t_stage3_us", "bytes_packed", "bytes_wire", "bytes_unpacked",
]


def _parse_size(text: str) -> GlobalGrid:
    parts = [int(x) for x in text.split(",")]
    if len(parts) == 1:
        parts = parts * 3
    if len(parts) != 3:
        raise argparse.ArgumentTypeError(f"--size wants 'n' or 'n0,n1,n2', got {text!r}")
    return GlobalGrid(*parts)


def _parse_procs(text: str) -> list[int]:
    try:
        procs = [int(x) for x in text.split(",")]
    except ValueError:
        raise argparse.ArgumentTypeError(f"--procs wants a comma list of ints, got {text!r}")
    if not procs or any(p < 1 for p in procs):
        raise argparse.ArgumentTypeError(f"--procs entries must be >= 1, got {text!r}")
    return procs


def _random_field(grid: GlobalGrid, seed: int) -> torch.Tensor:
    """Seeded standard-normal field (numpy default_rng, as cli.py:78-80)."""
    import numpy as np

    return torch.from_numpy(np.random.default_rng(seed).standard_normal((grid.n0, grid.n1, grid.n2)))


def _dft3d_r2c(field: torch.Tensor) -> torch.Tensor:
    """Direct triple-sum half spectrum (oracle.py:30-45), float64 on the device."""
    n0, n1, n2 = field.shape
    dev = torch.device("cuda", torch.cuda.current_device())

    def basis(n, m):
        k = torch.arange(m, dtype=torch.float64, device=dev)[:, None]
        j = torch.arange(n, dtype=torch.float64, device=dev)[None, :]
        return torch.exp(-2j * math.pi * (k * j) / n)

    f = field.to(dev, torch.complex128)
    return torch.einsum("ai,bj,ck,ijk->abc", basis(n0, n0), basis(n1, n1), basis(n2, n2 // 2 + 1), f)


def _verify_grids(max_size: int) -> list[GlobalGrid]:
    grids, s = [], 2
    while s <= max_size:
        grids.append(GlobalGrid(s, s, s))
        s *= 2
    if max_size >= 8:
        grids += [GlobalGrid(4, 8, 4), GlobalGrid(8, 4, 2)]
    return grids


def _parse_strategies(text: str) -> list[Strategy]:
    if text == "both":
        return [Strategy.STRIDED, Strategy.TRANSPOSE]
    return [Strategy(text)]


def _run_pipeline(grid: GlobalGrid, p: int, field: torch.Tensor, iters: int = 0, warmup: int = 0,
                  strategy: Strategy = Strategy.STRIDED, pattern: CommPattern = CommPattern.PAIRWISE):
    """forward (+ inverse pairs when timing) on p ranks; returns the gathered
    spectrum, per-iteration records (wall us, stage dict, counters) merged
    over ranks, and the worst round-trip relative rms (cli.py:87-128)."""
    slabs = scatter_real(field, grid, p)

    def body(ep):
        fp = plan(grid, ep, strategy, pattern, check_consistency=True)
        fp.enable_timing(True)
        mine = slabs[ep.rank]
        recs = []
        for _ in range(warmup + iters):
            fp.reset_instrumentation()
            ep.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            inverse(fp, forward(fp, mine))
            e1.record()
            ep.barrier()
            recs.append((e0.elapsed_time(e1) * 1e3, dict(fp.timers_us), fp.counters.snapshot()))
        spec = forward(fp, mine)
        kept = SpectralSlab(spec.layout, spec.tag, spec.data.clone())
        out = inverse(fp, spec)
        rel = (torch.linalg.norm(out.data - mine.data) / torch.linalg.norm(mine.data)).item()
        back = RealSlab(out.layout, out.data.clone())
        fp.close()
        return recs[warmup:], kept, rel, back

    per_rank = run_spmd(p, body)
    gathered = gather_spectral([r[1] for r in per_rank])
    merged = []
    for it in range(iters):
        wall = max(r[0][it][0] for r in per_rank)
        stages = {k: max(r[0][it][1][k] for r in per_rank) for k in ("stage1_us", "exchange_us", "stage3_us")}
        counters = tuple(sum(r[0][it][2][i] for r in per_rank) for i in range(3))
        merged.append((wall, stages, counters))
    return gathered, merged, max(r[2] for r in per_rank)


def _check(report, failures, grid, p, strategy, name, err, tol):
    status = "PASS" if err <= tol else "FAIL"
    line = (f"{grid.n0}x{grid.n1}x{grid.n2} p={p} {strategy:9s} {name:22s} "
            f"max_error={err:.3e} (tol {tol:.1e}) {status}")
    report.append(line)
    if status == "FAIL":
        failures.append(line)


def cmd_verify(args) -> int:
    if args.max_size > MAX_VERIFY_SIZE:
        print(f"usage error: --max-size is capped at {MAX_VERIFY_SIZE} (brute-force oracle cost)")
        return 2
    for p in args.procs:
        validate(GlobalGrid(args.max_size, args.max_size, args.max_size), p)
    report, failures, checks = [], [], 0
    for grid in _verify_grids(args.max_size):
        field = _random_field(grid, args.seed)
        ref = _dft3d_r2c(field).cpu().numpy()
        for p in args.procs:
            try:
                validate(grid, p)
            except ConfigurationError:
                continue
            spectra = {}
            for strategy in args.strategies:
                gathered, _, rel = _run_pipeline(grid, p, field, strategy=strategy, pattern=args.comm)
                spectra[strategy] = gathered
                for name, err, tol in (("oracle_equivalence", float(abs(gathered - ref).max()), ORACLE_ATOL),
                                       ("round_trip", rel, ROUNDTRIP_RTOL)):
                    _check(report, failures, grid, p, strategy.value, name, err, tol)
                    checks += 1
            if len(spectra) == 2:
                a = spectra[Strategy.STRIDED].view("float64")
                b = spectra[Strategy.TRANSPOSE].view("float64")
                diff = 0.0 if (a == b).all() else float(abs(a - b).max())
                _check(report, failures, grid, p, "both", "strategy_equivalence", diff, 0.0)
                checks += 1
    for line in report:
        print(line)
    print(f"{checks} checks, {len(failures)} failures")
    return 0 if not failures else 1


def _bench_rows(grid: GlobalGrid, p: int, strategy: Strategy, args) -> list[dict]:
    field = _random_field(grid, args.seed)
    _, merged, rel = _run_pipeline(grid, p, field, args.iters, args.warmup, strategy, args.comm)
    if rel > ROUNDTRIP_RTOL:
        raise SlabFftError(f"embedded correctness cross-check failed: round-trip error {rel:.3e} "
                           f"exceeds {ROUNDTRIP_RTOL:.1e} on {grid.n0}x{grid.n1}x{grid.n2}, p={p}")
    rows = []
    for it, (wall, st, cnt) in enumerate(merged):
        rows.append({"grid_n0": grid.n0, "grid_n1": grid.n1, "grid_n2": grid.n2, "p": p,
                     "strategy": strategy.value, "comm_pattern": args.comm.value, "iter": it,
                     "t_total_us": f"{wall:.3f}", "t_stage1_us": f"{st['stage1_us']:.3f}",
                     "t_exchange_us": f"{st['exchange_us']:.3f}", "t_stage3_us": f"{st['stage3_us']:.3f}",
                     "bytes_packed": cnt[0], "bytes_wire": cnt[1], "bytes_unpacked": cnt[2]})
    med = statistics.median(float(r["t_total_us"]) for r in rows)
    print(f"grid {grid.n0}x{grid.n1}x{grid.n2}  p={p}  {strategy.value}  comm={args.comm.value}  mode={args.mode}  "
          f"iters={args.iters}  median pair {med:.1f} us", file=sys.stderr)
    return rows


def cmd_bench(args) -> int:
    if args.iters < 1:
        print("usage error: --iters must be >= 1")
        return 2
    grid = args.size
    rows = []
    for p in args.procs:
        validate(grid, p)
        for strategy in args.strategies:
            rows += _bench_rows(grid, p, strategy, args)
    out = open(args.output, "w", newline="") if args.output else sys.stdout
    writer = csv.DictWriter(out, fieldnames=CSV_COLUMNS)
    writer.writeheader()
    writer.writerows(rows)
    if args.output:
        out.close()
    return 0


def cmd_compare(args) -> int:
    """Both strategies on identical inputs (cli.py:342-383)."""
    if args.iters < 1:
        print("usage error: --iters must be >= 1")
        return 2
    grid = args.size
    field = _random_field(grid, args.seed)
    status = 0
    for p in args.procs:
        validate(grid, p)
        res = {}
        for strategy in (Strategy.STRIDED, Strategy.TRANSPOSE):
            gathered, merged, rel = _run_pipeline(grid, p, field, args.iters, args.warmup, strategy, args.comm)
            if rel > ROUNDTRIP_RTOL:
                raise SlabFftError(f"round-trip error {rel:.3e} exceeds {ROUNDTRIP_RTOL:.1e} for {strategy.value}")
            res[strategy] = (gathered, merged)
        print(f"grid {grid.n0}x{grid.n1}x{grid.n2}  p={p}  comm={args.comm.value}  mode={args.mode}  iters={args.iters}")
        print(f"{'strategy':10s} {'t_total_us(med)':>16s} {'t_exchange_us(med)':>19s} "
              f"{'packed':>12s} {'wire':>12s} {'unpacked':>12s}")
        totals = {}
        for strategy, (_, merged) in res.items():
            tot = statistics.median(m[0] for m in merged)
            exch = statistics.median(m[1]["exchange_us"] for m in merged)
            cnt = merged[-1][2]
            totals[strategy] = (tot, sum(cnt))
            print(f"{strategy.value:10s} {tot:16.1f} {exch:19.1f} {cnt[0]:12d} {cnt[1]:12d} {cnt[2]:12d}")
        s_bytes, t_bytes = totals[Strategy.STRIDED][1], totals[Strategy.TRANSPOSE][1]
        if s_bytes > 0:
            print(f"copy-byte ratio transpose/strided: {t_bytes / s_bytes:.2f}")
        else:
            print("copy-byte ratio transpose/strided: n/a (no exchanged bytes at p=1)")
        t_t, t_s = totals[Strategy.TRANSPOSE][0], totals[Strategy.STRIDED][0]
        print(f"median pair time: strided {100.0 * (t_t - t_s) / t_t:+.1f}% vs transpose (B200, device-timed)")
        same = (res[Strategy.STRIDED][0].view("float64") == res[Strategy.TRANSPOSE][0].view("float64")).all()
        print(f"spectra bitwise identical: {'yes' if same else 'NO'}")
        if not same:
            status = 1
    return status


def _add_common(sub, default_mode: str) -> None:
    """--comm / --mode / --seed as in cli.py:390-396.  --mode is accepted for
    command-line compatibility only: GPU ranks always run as concurrent host
    threads (the reference's SERIAL turnstile is a scheduling device of its
    simulated fabric)."""
    sub.add_argument("--comm", type=CommPattern, choices=list(CommPattern), default=CommPattern.PAIRWISE, metavar="{pairwise,collective}",
                     help="all-to-all pattern: pairwise or collective (default pairwise)")
    sub.add_argument("--mode", choices=["threaded", "serial"], default=default_mode,
                     help="accepted for compatibility; ranks always run as threads")
    sub.add_argument("--seed", type=int, default=0)


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_1406_5597_b200",
                                     description="B200 transpose-free slab 3D FFT: verification and benchmarks.")
    sub = parser.add_subparsers(dest="command", required=True)
    pv = sub.add_parser("verify", help="oracle-equivalence and round-trip suites")
    pv.add_argument("--max-size", type=int, default=8)
    pv.add_argument("--procs", type=_parse_procs, default=[1, 2, 4])
    pv.add_argument("--strategy", dest="strategies", type=_parse_strategies,
                    default=[Strategy.STRIDED, Strategy.TRANSPOSE])
    _add_common(pv, "serial")
    pv.set_defaults(func=cmd_verify)
    pb = sub.add_parser("bench", help="time forward+inverse pairs and emit CSV")
    pb.add_argument("--size", type=_parse_size, required=True)
    pb.add_argument("--procs", type=_parse_procs, default=[1])
    pb.add_argument("--iters", type=int, default=5)
    pb.add_argument("--warmup", type=int, default=1)
    pb.add_argument("--output", default=None)
    pb.add_argument("--strategy", dest="strategies", type=_parse_strategies, default=[Strategy.STRIDED])
    _add_common(pb, "threaded")
    pb.set_defaults(func=cmd_bench)
    pc = sub.add_parser("compare", help="run both strategies on identical inputs")
    pc.add_argument("--size", type=_parse_size, required=True)
    pc.add_argument("--procs", type=_parse_procs, default=[4])
    pc.add_argument("--iters", type=int, default=5)
    pc.add_argument("--warmup", type=int, default=1)
    _add_common(pc, "threaded")
    pc.set_defaults(func=cmd_compare)
    return parser


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return int(exc.code or 0)
    try:
        return args.func(args)
    except ConfigurationError as exc:
        print(f"configuration error: {exc}")
        return 2
    except OSError as exc:
        print(f"I/O error: {exc}")
        return 2
    except SlabFftError as exc:
        print(f"check failure: {exc}")
        return 1
