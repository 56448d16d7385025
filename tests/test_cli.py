"""CLI parity with the reference tool (cli.py): exit codes on CPU, suites on GPU."""

import csv
import io
import sys

import pytest

from paper_1406_5597_b200 import cli


def test_usage_errors_exit_2():
    assert cli.main(["verify", "--max-size", "64"]) == 2          # cli.py:160-162
    assert cli.main(["verify", "--max-size", "8", "--procs", "3"]) == 2  # p does not divide
    assert cli.main(["bench", "--size", "8", "--iters", "0"]) == 2
    assert cli.main(["compare", "--size", "8", "--iters", "0"]) == 2
    assert cli.main(["nonsense"]) == 2


def test_csv_header_matches_reference():
    assert cli.CSV_COLUMNS == [
        "grid_n0", "grid_n1", "grid_n2", "p", "strategy", "comm_pattern", "iter", "t_total_us",
        "t_stage1_us", "t_exchange_us", "t_stage3_us", "bytes_packed", "bytes_wire", "bytes_unpacked"]


@pytest.mark.gpu
def test_verify_suites_pass(capsys):
    assert cli.main(["verify", "--max-size", "8", "--procs", "1,2,4"]) == 0
    out = capsys.readouterr().out
    assert "0 failures" in out and "FAIL" not in out


@pytest.mark.gpu
def test_bench_csv(tmp_path):
    path = tmp_path / "b.csv"
    assert cli.main(["bench", "--size", "16", "--procs", "1,2", "--iters", "2", "--warmup", "1",
                     "--output", str(path)]) == 0
    rows = list(csv.DictReader(open(path)))
    assert len(rows) == 4
    for r in rows:
        assert r["strategy"] == "strided" and int(r["bytes_packed"]) == 0 and int(r["bytes_unpacked"]) == 0
        p = int(r["p"])
        # wire bytes per pair, summed over ranks: 2 * p * (p-1) * n0p * n1p * n2c * 16
        assert int(r["bytes_wire"]) == 2 * p * (p - 1) * (16 // p) * (16 // p) * 9 * 16


@pytest.mark.gpu
def test_compare_strategies(capsys):
    assert cli.main(["compare", "--size", "32", "--procs", "2,4", "--iters", "2"]) == 0
    out = capsys.readouterr().out
    assert out.count("spectra bitwise identical: yes") == 2
    assert out.count("copy-byte ratio transpose/strided: 3.00") == 2
