"""bench.py --fmbench: the reference harness's bench / verify / memory reports
(proj/src/bench.cpp:62-209, 298-346; CLI proj/tools/fmbench.cpp:36-68) with the
GPU route as an extra `cuda` row / column, in the reference's CSV schema
(tests/golden/bench_columns.txt, tests/golden/memory_f32_k4_12.csv)."""
import csv
import io
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"


def _run(*args, timeout=600):
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--fmbench", *args], capture_output=True,
                       text=True, timeout=timeout, cwd=ROOT)
    return p.returncode, p.stdout


def _csv(text):
    return list(csv.reader(io.StringIO("\n".join(ln for ln in text.splitlines() if ln and not ln.startswith("#")))))


def test_config_validation_reports_error():
    # bench.cpp:230-240 messages; the report carries the error, exit status 2
    rc, out = _run("bench", "--k-start", "0")
    assert rc == 2 and "# bench: ERROR k-start must be at least 1" in out
    rc, out = _run("verify", "--k-start", "30", "--k-stop", "20")
    assert rc == 2 and "verify: ERROR at k-start must not exceed k-stop" in out
    rc, out = _run("memory", "--sigma", "0")
    assert rc == 2 and "sigma must be positive" in out


def test_memory_model_matches_golden_table():
    # proj/tests/golden/memory_f32_k4_12.csv; --mem-cap-bytes 0 keeps every row
    # model-only (no solver cross-check), so this runs without a GPU
    rc, out = _run("memory", "--k-start", "4", "--k-stop", "12", "--k-step", "4", "--precision", "f32",
                   "--mem-cap-bytes", "0")
    assert rc == 0, out
    rows = _csv(out)
    gold = [r for r in csv.reader(open(GOLDEN / "memory_f32_k4_12.csv")) if r and not r[0].startswith("#")]
    assert rows[0][:5] == gold[0] and rows[0][5] == "cuda_peak_extra_bytes"
    assert [r[:5] for r in rows[1:]] == gold[1:]
    assert all(r[5] == "" for r in rows[1:])


@pytest.mark.gpu
def test_bench_csv_has_reference_schema_and_cuda_rows():
    rc, out = _run("bench", "--k-start", "8", "--k-stop", "40", "--k-step", "16", "--batch", "3", "--reps", "2",
                   "--warmup", "1", "--precision", "f32", "--mask", "resolvent")
    assert rc == 0, out
    assert out.startswith("# functional-map solver benchmark")
    rows = _csv(out)
    assert ",".join(rows[0]) == open(GOLDEN / "bench_columns.txt").read().strip()
    body = rows[1:]
    assert [(r[0], r[1]) for r in body] == [(str(k), s) for k in (8, 24, 40) for s in ("rowwise", "batched", "cuda")]
    for r in body:
        assert r[6] == "ok"
        assert float(r[2]) > 0 and int(r[4]) >= 0 and float(r[5]) > 0
        if r[1] == "cuda":
            assert float(r[3]) <= 1e-3  # f32 route vs the f32 rowwise reference (bench.cpp:28 tolerance)


@pytest.mark.gpu
def test_bench_mem_cap_skips_batched_row_only():
    rc, out = _run("bench", "--k-start", "16", "--k-stop", "16", "--reps", "1", "--warmup", "0", "--precision",
                   "f32", "--mem-cap-bytes", "1000")
    assert rc == 0, out
    rows = {r[1]: r for r in _csv(out)[1:]}
    assert rows["batched"][6] == "mem-cap-skipped" and rows["batched"][4] == str(16 ** 3 * 4)
    assert rows["rowwise"][6] == "ok"


@pytest.mark.gpu
def test_verify_passes_and_catches_injected_fault():
    # f64 (the reference default): the k^2 x k^2 oracle runs for k <= 32 (in f32 it
    # is numerically singular from k ~ 24 on, as in the reference); at --precision
    # f64 the cuda route is fmap_solve_f64 (f64 end to end) and is held to 1e-8
    rc, out = _run("verify", "--k-start", "12", "--k-stop", "36", "--k-step", "12", "--batch", "2", "--precision",
                   "f64")
    assert rc == 0, out
    assert "rowwise~cuda=" in out and "cuda~oracle=" in out and "verify: PASS" in out
    rc, out = _run("verify", "--k-start", "12", "--k-stop", "12", "--batch", "2", "--precision", "f32",
                   "--inject-fault")
    assert rc == 1 and "verify: FAIL" in out


@pytest.mark.gpu
def test_memory_reports_cuda_route_bytes():
    rc, out = _run("memory", "--k-start", "4", "--k-stop", "12", "--k-step", "4", "--precision", "f32")
    assert rc == 0, out
    rows = _csv(out)[1:]
    gold = [r for r in csv.reader(open(GOLDEN / "memory_f32_k4_12.csv")) if r and not r[0].startswith("#")]
    assert [r[:5] for r in rows] == gold[1:]
    assert all(int(r[5]) > 0 for r in rows)
