"""bench.py's JSON contract (the driver parses one line per run).  The
reference arm runs on the CPU here; the GPU arm runs on the B200 box."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    """--impl reference: the oracle port timed on the host cores, same metric
    and unit as the GPU arm, plus cpu_baseline and a zero-copy e2e."""
    d = _run(["--impl", "reference", "--grid", "32", "--steps", "1", "--warmup", "0", "--cpu-planes", "8"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["unit"] == "GFLOP/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    # the GPU arm's workload string, so the driver's ratio compares like with like
    assert d["config"]["workload"] == "32x32x32 float64 r2c+c2r pair, slab p=1"
    assert d["config"]["parallelism"] == "slab1"
    # measured, not extrapolated: the timed steps are the reported step time
    assert len(d["cpu_baseline"]["timed_steps_s"]) == 1
    assert abs(d["cpu_baseline"]["timed_steps_s"][0] * 1e3 - d["ms_per_step"]) < 1.0 + 1e-3 * d["ms_per_step"]


def test_reference_arm_config_matches_gpu_arm():
    """Both arms print the same config object (bench.cube_config), key for key."""
    import bench

    d = _run(["--impl", "reference", "--grid", "32", "--steps", "1", "--warmup", "0", "--cpu-planes", "8"])
    assert d["config"] == bench.cube_config(32, 32, 32, "float64", 1)


def test_gpus_n_without_torchrun_self_launches(monkeypatch):
    """--gpus N > 1 outside torchrun re-executes itself under torch.distributed.run."""
    import bench

    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    assert bench.main() == 0
    cmd = calls[0]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]


def test_stage3_kernel_name_follows_the_library_defaults(monkeypatch):
    """roofline.kernel names the stage-3 kernel libtffft runs by default
    (columns_wpc / columns_tma in csrc/tffft.cu): float64 1024-point columns
    keep col_tma_kernel, 512-point / float32 1024-point columns the
    warp-per-column kernel, 2048-point columns its tensor-memory 2 x 1024
    variant, other lengths col_fft_kernel; TFFFT_WPC / TFFFT_TMA_COLS override."""
    import bench

    monkeypatch.delenv("TFFFT_WPC", raising=False)
    monkeypatch.delenv("TFFFT_TMA_COLS", raising=False)
    assert bench.stage3_kernel_name(1024, "float64") == "col_tma_kernel"
    assert bench.stage3_kernel_name(1024, "float32") == "col_wpc_kernel"
    assert bench.stage3_kernel_name(512, "float64") == "col_wpc_kernel"
    assert bench.stage3_kernel_name(2048, "float64") == "col_wpc2_kernel"
    assert bench.stage3_kernel_name(256, "float64") == "col_fft_kernel"
    monkeypatch.setenv("TFFFT_WPC", "1")
    assert bench.stage3_kernel_name(1024, "float64") == "col_wpc_kernel"
    monkeypatch.setenv("TFFFT_WPC", "0")
    assert bench.stage3_kernel_name(512, "float64") == "col_tma_kernel"
    assert bench.stage3_kernel_name(2048, "float64") == "col_fft_kernel"
    monkeypatch.setenv("TFFFT_TMA_COLS", "0")
    assert bench.stage3_kernel_name(1024, "float64") == "col_fft_kernel"


@pytest.mark.gpu
def test_gpu_arm_line():
    """The GPU arm at a small grid: device-timed value, roofline with the
    stage-3 kernel, host-buffer e2e, launch count, clocks, cpu_baseline."""
    d = _run(["--grid", "128", "--steps", "3", "--warmup", "3", "--e2e-steps", "2", "--cpu-planes", "8"])
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["details"]["roundtrip_rel_l2"] <= 1e-12
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.5 and r["unit"] == "GB/s"
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 128 ** 3 * 8 and e["d2h_bytes_per_step"] == 128 ** 3 * 8
    assert d["gpu_launches"] == 7 * 3  # six FFT kernels + the consistency reduction per pair
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["cpu_baseline"]["value"] > 0
