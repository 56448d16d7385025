"""Time ONE full-size forward + inverse pair of the oracle port (bit-identical
to the reference STRIDED path, dfft.py:148-215) on all host cores, at p = 1,
and write the measurement as JSON (profiles/r02_cpu_full_pair.json).

This is the measured CPU number beside bench.py's bounded per-step sample
(bench.cpu_sample); run it on the GPU host:

    python tools/cpu_full_pair.py --grid 1024 --out profiles/r02_cpu_full_pair.json
"""

import argparse
import json
import math
import os
import platform
import resource
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=1024)
    ap.add_argument("--seed", type=int, default=11)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    n = a.grid
    shape = (n, n, n)
    workers = len(os.sched_getaffinity(0))
    x = oracle.uniform_field(shape, a.seed)
    t0 = time.perf_counter()
    flats = oracle.forward_all(x, 1, workers=workers)
    t1 = time.perf_counter()
    outs, res = oracle.inverse_all(flats, shape, workers=workers)
    t2 = time.perf_counter()
    err = float(np.linalg.norm(outs[0].reshape(-1) - x.reshape(-1)) / np.linalg.norm(x.reshape(-1)))
    N = n ** 3
    flops = 2 * 2.5 * N * math.log2(N)
    rec = {
        "what": "oracle port (bit-identical to the reference STRIDED path), one full forward + inverse pair, p=1",
        "grid": [n, n, n], "dtype": "float64", "threads": workers, "cpu": cpu_model(),
        "forward_s": round(t1 - t0, 3), "inverse_s": round(t2 - t1, 3), "pair_s": round(t2 - t0, 3),
        "gflops": flops / (t2 - t0) / 1e9, "roundtrip_rel_l2": err, "imag_residue": res,
        "max_rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6,
        "reference_single_core_pair_s": 447.6 if n == 1024 else None,
        "note": "the unmodified reference (pure Python + numpy, ~1-2 cores under the GIL) took 447.6 s per "
                "1024^3 pair in the survey's measurement (BASELINE.md §2); this port batches rows across threads",
    }
    line = json.dumps(rec)
    print(line)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
