"""report/trace CSV and CLI parity with the reference.

The reference's writers (harness.py:299-334) and CLI (cli.py:15-86) define
formats "so reports diff cleanly".  Here the STOCK reference (oracle/_ref,
engine "native") and this package (CUDA) run the same benchmark; the CSV files
must be identical except the timing columns (seconds, teps, layer elapsed),
and the stock writer applied to this package's report must reproduce this
package's file byte for byte."""

from __future__ import annotations

import csv
import io
import os
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu

TIMED_REPORT = {"seconds", "teps"}
TIMED_TRACE = {"elapsed", "seconds"}


@pytest.fixture(scope="module")
def stock(cuda):
    from oracle import refpkg

    hybfs = refpkg.load()
    assert hybfs is not None, "oracle/_ref must ship the stock hybfs package"
    return hybfs


def masked(path, timed):
    """(comment lines, header, rows with the timing columns blanked)."""
    with open(path, encoding="utf-8") as fh:
        text = fh.read()
    assert "\r" not in text
    lines = text.split("\n")
    comments = [x for x in lines if x.startswith("#")]
    body = "\n".join(x for x in lines if not x.startswith("#"))
    rows = list(csv.reader(io.StringIO(body)))
    head = rows[0]
    idx = [i for i, h in enumerate(head) if h in timed]
    out = [[("*" if i in idx else c) for i, c in enumerate(r)] for r in rows[1:]]
    return comments, head, out


@pytest.mark.parametrize("mode", ["simd-hybrid", "scalar-hybrid", "scalar-td", "scalar-bu"])
def test_report_and_trace_csv_match_reference(cuda, stock, tmp_path, mode):
    hb = cuda
    params_kw = dict(scale=11, edgefactor=16, seed=3)
    ref = stock.harness.run_benchmark(stock.generator.GraphParams(**params_kw), mode=mode, runs=16,
                                      engine_name="native")
    ours = hb.run_benchmark(hb.GraphParams(**params_kw), mode=mode, runs=16)
    files = {}
    for who, rep, mod in (("ref", ref, stock.harness), ("ours", ours, hb.harness)):
        files[who] = (tmp_path / f"{who}_report.csv", tmp_path / f"{who}_trace.csv")
        mod.write_report_csv(rep, files[who][0])
        mod.write_trace_csv(rep, files[who][1])
    assert masked(files["ref"][0], TIMED_REPORT) == masked(files["ours"][0], TIMED_REPORT)
    assert masked(files["ref"][1], TIMED_TRACE) == masked(files["ours"][1], TIMED_TRACE)
    # the stock writers on our report: byte-identical to our writers
    stock.harness.write_report_csv(ours, tmp_path / "x_report.csv")
    stock.harness.write_trace_csv(ours, tmp_path / "x_trace.csv")
    assert (tmp_path / "x_report.csv").read_bytes() == files["ours"][0].read_bytes()
    assert (tmp_path / "x_trace.csv").read_bytes() == files["ours"][1].read_bytes()
    assert ours.teps_denominator == ref.teps_denominator
    assert [r.source for r in ours.runs] == [r.source for r in ref.runs]
    assert all(r.valid for r in ours.runs)


def test_cli_end_to_end_matches_reference_cli(cuda, stock, tmp_path):
    """`python -m paper_1704_02259_b200.cli` on the GPU (--gpus 1, --out,
    --trace-out, --csr-cache, run twice so the second run loads the cache)
    against the stock CLI's files for the same flags."""
    from oracle import refpkg

    common = ["--scale", "10", "--edgefactor", "16", "--seed", "2", "--mode", "simd-hybrid",
              "--alpha", "14", "--beta", "24", "--runs", "12"]
    ref_dir = refpkg.package_dir()
    r = subprocess.run([sys.executable, "-c", "import sys; from hybfs.cli import main; sys.exit(main())",
                        *common, "--out", str(tmp_path / "r.csv"), "--trace-out", str(tmp_path / "rt.csv")],
                       env={**os.environ, "PYTHONPATH": ref_dir}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "engine in use: native" in r.stdout
    cache = tmp_path / "g.csr"
    for attempt in range(2):
        o = subprocess.run([sys.executable, "-m", "paper_1704_02259_b200.cli", *common, "--gpus", "1",
                            "--out", str(tmp_path / "o.csv"), "--trace-out", str(tmp_path / "ot.csv"),
                            "--csr-cache", str(cache)],
                           cwd=REPO, capture_output=True, text=True, timeout=600)
        assert o.returncode == 0, o.stdout[-2000:] + o.stderr[-2000:]
        assert cache.exists()
        assert masked(tmp_path / "r.csv", TIMED_REPORT) == masked(tmp_path / "o.csv", TIMED_REPORT)
        assert masked(tmp_path / "rt.csv", TIMED_TRACE) == masked(tmp_path / "ot.csv", TIMED_TRACE)
