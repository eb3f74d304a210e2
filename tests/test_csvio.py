"""CSV matrix I/O (paper_2604_10377_b200/csvio.py) — the reference's csv.cpp
contract, cases restated from proj/tests/test_csv.cpp (line cited per test).
Host-only: runs without a GPU."""
import io
import math

import numpy as np
import pytest

from paper_2604_10377_b200 import csvio


def test_reading_a_plain_matrix():
    # test_csv.cpp:11-22
    m = csvio.read_matrix_csv(io.StringIO("1,2.5,-3\n4e2, 0.125 ,6\n"))
    assert m.shape == (2, 3)
    assert m.tolist() == [[1.0, 2.5, -3.0], [400.0, 0.125, 6.0]]


def test_ragged_rows_are_rejected():
    # test_csv.cpp:24-33
    with pytest.raises(RuntimeError) as ei:
        csvio.read_matrix_csv(io.StringIO("1,2\n3\n"))
    assert "line 2" in str(ei.value) and "ragged" in str(ei.value)


@pytest.mark.parametrize("text", ["1,2\n3,x\n", "1,2\n3,4junk\n", "1,\n", "+1\n", "1_0\n", "0x10\n", " \n"])
def test_garbage_cells_are_rejected(text):
    # test_csv.cpp:35-42, plus from_chars strictness (no '+', separators, hex; a
    # whitespace-only line is one empty cell)
    with pytest.raises(RuntimeError):
        csvio.read_matrix_csv(io.StringIO(text))


def test_empty_input_is_rejected():
    # test_csv.cpp:44-47
    with pytest.raises(RuntimeError, match="no rows"):
        csvio.read_matrix_csv(io.StringIO(""))


def test_blank_lines_and_crlf_are_skipped():
    # test_csv.cpp:49-53 (+ Windows line ends: csv.cpp trims a trailing '\r')
    assert csvio.read_matrix_csv(io.StringIO("\n1,2\n\n3,4\n\n")).shape == (2, 2)
    assert csvio.read_matrix_csv(io.StringIO("1,2\r\n3,4\r\n")).tolist() == [[1.0, 2.0], [3.0, 4.0]]


def test_missing_files_are_reported():
    # test_csv.cpp:55-57
    with pytest.raises(RuntimeError, match="cannot open"):
        csvio.read_matrix_csv("/nonexistent/matrix.csv")


def test_17_significant_digits_round_trip_exactly(tmp_path):
    # test_csv.cpp:59-78 (seeded numpy stand-in for the mt19937_64 draw)
    rng = np.random.default_rng(2024)
    m = rng.standard_normal((4, 4)) * 10.0 ** (np.arange(16).reshape(4, 4) - 8)
    m[0, :] = [1.0 / 3.0, 3.141592653589793, 1e-300, 0.0]
    buf = io.StringIO()
    csvio.write_matrix_csv(buf, m, 17)
    back = csvio.read_matrix_csv(io.StringIO(buf.getvalue()))
    assert back.shape == m.shape and np.array_equal(back, m)
    p = tmp_path / "m.csv"
    csvio.write_matrix_csv(p, m)
    assert np.array_equal(csvio.read_matrix_csv(p), m)


def test_format_value_round_trips_individual_doubles():
    # test_csv.cpp:80-88
    for v in (2.0 / 3.0, 1.0000000000000002, -9.87e123, 5e-324):
        assert float(csvio.format_value(v, 17)) == v
    assert csvio.format_value(0.1, 9) == "0.100000001" or csvio.format_value(0.1, 9) == "0.1"


def test_special_values_parse_like_from_chars():
    m = csvio.read_matrix_csv(io.StringIO("inf,-INFINITY,nan\n"))
    assert m[0, 0] == math.inf and m[0, 1] == -math.inf and math.isnan(m[0, 2])


@pytest.mark.gpu
def test_file_loaded_descriptors_through_the_gpu_route(tmp_path, fm, oracle):
    # SPEC "External Interfaces": descriptors / mask as CSV files -> solve -> C as CSV
    k, d = 30, 60
    _, _, M, a, b = oracle.random_problem(k, d, 77, kind=1)
    for name, x in (("a", a), ("b", b), ("m", M)):
        csvio.write_matrix_csv(tmp_path / f"{name}.csv", x)
    A, B, Mm = (csvio.read_matrix_csv(tmp_path / f"{n}.csv") for n in ("a", "b", "m"))
    rep = fm.solve_cuda(A, B, Mm, 100.0)
    csvio.write_matrix_csv(tmp_path / "c.csv", rep.map, 9)
    C = csvio.read_matrix_csv(tmp_path / "c.csv")
    G, R = oracle.normal_equations(a, b)
    ref = oracle.solve(G, R, M, 100.0, route="batched", dtype=np.float32)
    assert np.abs(C - ref.maps).max() <= 1e-4 * np.abs(ref.maps).max()
