"""CSV matrix format shared by the reference's tools (SPEC.md "External
Interfaces": one row per line, comma-separated decimal floats, no header;
ragged rows rejected) — restates /root/reference/proj/src/csv.cpp:13-92:

  read_matrix_csv(path | text stream) -> float64 [rows, cols]   (csv.cpp:30-70)
  write_matrix_csv(path | stream, m, significant_digits=17)     (csv.cpp:77-92)
  format_value(v, significant_digits) -> "%.*g"                 (csv.cpp:71-75)

Cells are parsed like std::from_chars(double) after trimming spaces / tabs (and a
trailing '\\r'): plain or exponent decimal notation, optional leading '-', "inf" /
"infinity" / "nan" spellings; no leading '+', no digit separators, no hex.
Errors raise CsvError (a RuntimeError, like the reference's std::runtime_error)
naming the 1-based line.  These matrices feed the GPU entry points as host
arrays (e.g. descriptors A, B -> fmsolve.normal_equations / solve_host).
"""
from __future__ import annotations

import io
import os
import re
from typing import IO, Union

import numpy as np

__all__ = ["CsvError", "read_matrix_csv", "write_matrix_csv", "format_value"]

# std::from_chars(double, chars_format::general): [-] (digits [. digits] | . digits) [(e|E) [+|-] digits],
# or inf / infinity / nan / nan(chars), case-insensitive
_DECIMAL = re.compile(
    r"-?(?:(?:[0-9]+(?:\.[0-9]*)?|\.[0-9]+)(?:[eE][+-]?[0-9]+)?|(?i:inf(?:inity)?|nan(?:\([0-9A-Za-z_]*\))?))")


class CsvError(RuntimeError):
    pass


def _parse_cell(cell: str, line_number: int) -> float:
    s = cell.strip(" \t")
    if s.endswith("\r"):
        s = s[:-1].rstrip(" \t")
    if not s or not _DECIMAL.fullmatch(s):
        raise CsvError(f"line {line_number}: cannot parse '{cell}' as a decimal float")
    low = s.lower().lstrip("-")
    if low.startswith("nan"):
        return float("-nan") if s.startswith("-") else float("nan")
    return float(s)


def read_matrix_csv(src: Union[str, os.PathLike, IO[str]]) -> np.ndarray:
    """csv.cpp:30-70 (stream) and :63-68 (path)."""
    if isinstance(src, (str, os.PathLike)):
        try:
            f = open(src, "r", newline="")
        except OSError:
            raise CsvError(f"cannot open '{os.fspath(src)}' for reading") from None
        with f:
            return read_matrix_csv(f)
    rows: list[list[float]] = []
    for line_number, raw in enumerate(src.read().split("\n"), start=1):
        line = raw
        if line == "" or line == "\r":
            continue
        row = [_parse_cell(c, line_number) for c in line.split(",")]
        if rows and len(row) != len(rows[0]):
            raise CsvError(f"line {line_number}: ragged row with {len(row)} cells, expected {len(rows[0])}")
        rows.append(row)
    if not rows:
        raise CsvError("matrix file holds no rows")
    return np.array(rows, dtype=np.float64)


def format_value(value: float, significant_digits: int) -> str:
    """csv.cpp:71-75: printf("%.*g")."""
    return "%.*g" % (significant_digits, value)


def write_matrix_csv(dst: Union[str, os.PathLike, IO[str]], m, significant_digits: int = 17) -> None:
    """csv.cpp:77-92."""
    a = np.asarray(m, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("write_matrix_csv needs a 2-D matrix")
    if isinstance(dst, (str, os.PathLike)):
        try:
            f = open(dst, "w", newline="")
        except OSError:
            raise CsvError(f"cannot open '{os.fspath(dst)}' for writing") from None
        with f:
            write_matrix_csv(f, a, significant_digits)
        return
    out = io.StringIO()
    for row in a:
        out.write(",".join(format_value(float(v), significant_digits) for v in row))
        out.write("\n")
    dst.write(out.getvalue())
