"""Exchange formats between the CPU oracle / reference and the B200 runs.

Byte-compatible restatements of the reference writers:
  * raw field: `<base>.bin` (x-fastest float64) + `<base>.json` header
    {dim, h, layout, n, t}  (write_field_binary, stencil_main.cpp:131-142);
  * MatrixMarket coordinate real general, 1-based, `%.17g` values
    (write_matrix_market, io.cpp:109-118);
  * CSV with `%.17g` values (write_csv, io.cpp:120-130).
Plus the readers the reference lacks (it only writes), so a field dumped by
either side can resume a run on the other.
"""
from __future__ import annotations

import json
from pathlib import Path
from typing import Sequence, Tuple

import numpy as np

from .errors import Errc, StencilkitError


def format_double(v: float) -> str:
    """%.17g (io.cpp:97-101)."""
    return "%.17g" % v


def write_field_binary(base: str | Path, field: np.ndarray, dim: int, n: Sequence[int], h: float, t: float = 0.0) -> None:
    base = Path(base)
    c = np.ascontiguousarray(field, dtype="<f8").ravel()
    if c.size != int(np.prod(n)):
        raise StencilkitError(Errc.shape_mismatch, "field length does not match n")
    base.with_suffix(".bin").write_bytes(c.tobytes())
    header = {"dim": int(dim), "n": [int(v) for v in n], "h": float(h), "t": float(t), "layout": "x-fastest float64"}
    base.with_suffix(".json").write_text(json.dumps(header, indent=2, sort_keys=True) + "\n")


def read_field_binary(base: str | Path) -> Tuple[np.ndarray, dict]:
    base = Path(base)
    header = json.loads(base.with_suffix(".json").read_text())
    if header.get("layout") != "x-fastest float64":
        raise StencilkitError(Errc.invalid_argument, f"unsupported field layout {header.get('layout')!r}")
    c = np.frombuffer(base.with_suffix(".bin").read_bytes(), dtype="<f8").copy()
    if c.size != int(np.prod(header["n"])):
        raise StencilkitError(Errc.shape_mismatch, "field file does not match its header")
    return c, header


def write_matrix_market(path: str | Path, row_ptr: np.ndarray, col_idx: np.ndarray, values: np.ndarray,
                        cols: int | None = None) -> None:
    rows = len(row_ptr) - 1
    cols = rows if cols is None else cols
    with open(path, "w", newline="\n") as out:
        out.write("%%MatrixMarket matrix coordinate real general\n")
        out.write(f"{rows} {cols} {len(values)}\n")
        for i in range(rows):
            for k in range(int(row_ptr[i]), int(row_ptr[i + 1])):
                out.write(f"{i + 1} {int(col_idx[k]) + 1} {format_double(float(values[k]))}\n")


def read_matrix_market(path: str | Path) -> Tuple[np.ndarray, np.ndarray, np.ndarray, int]:
    """Coordinate real general (as written above, rows in order) -> CSR."""
    with open(path) as f:
        if not f.readline().startswith("%%MatrixMarket matrix coordinate real general"):
            raise StencilkitError(Errc.invalid_argument, "not a coordinate real general MatrixMarket file")
        line = f.readline()
        while line.startswith("%"):
            line = f.readline()
        rows, cols, nnz = (int(v) for v in line.split())
        data = np.loadtxt(f, dtype=np.float64, ndmin=2) if nnz else np.zeros((0, 3))
    r = data[:, 0].astype(np.int64) - 1
    order = np.argsort(r, kind="stable")
    r, c, v = r[order], data[order, 1].astype(np.int64) - 1, data[order, 2]
    row_ptr = np.zeros(rows + 1, np.int64)
    np.add.at(row_ptr, r + 1, 1)
    return np.cumsum(row_ptr), c, v, cols


def write_csv(path: str | Path, header: Sequence[str], rows) -> None:
    with open(path, "w", newline="\n") as out:
        out.write(",".join(header) + "\n")
        for row in rows:
            out.write(",".join(format_double(float(x)) for x in row) + "\n")
