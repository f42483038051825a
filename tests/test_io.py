"""CPU: exchange formats (reference writers restated, plus readers)."""
from pathlib import Path

import numpy as np
import pytest

from paper_2205_03354_b200 import io
from paper_2205_03354_b200.errors import StencilkitError

GOLD = Path(__file__).resolve().parent / "golden"


def test_field_binary_round_trip(tmp_path):
    c = np.random.default_rng(0).uniform(-1, 1, 12 * 10)
    io.write_field_binary(tmp_path / "f", c, 2, [12, 10], 1 / 12, t=0.5)
    assert (tmp_path / "f.bin").read_bytes() == c.astype("<f8").tobytes()
    got, hdr = io.read_field_binary(tmp_path / "f")
    assert np.array_equal(got, c)
    assert hdr == {"dim": 2, "n": [12, 10], "h": 1 / 12, "t": 0.5, "layout": "x-fastest float64"}
    with pytest.raises(StencilkitError):
        io.write_field_binary(tmp_path / "g", c, 2, [5, 5], 0.1)


def test_matrix_market_round_trip(tmp_path):
    z = np.load(GOLD / "csr_bilap2d_cl17.npz")
    p = tmp_path / "m.mtx"
    io.write_matrix_market(p, z["row_ptr"], z["col_idx"], z["values"])
    lines = p.read_text().splitlines()
    assert lines[0] == "%%MatrixMarket matrix coordinate real general"
    rows = len(z["row_ptr"]) - 1
    assert lines[1] == f"{rows} {rows} {len(z['values'])}"
    first = lines[2].split()
    assert first[0] == "1" and int(first[1]) == z["col_idx"][0] + 1 and float(first[2]) == z["values"][0]
    rp, ci, v, cols = io.read_matrix_market(p)
    assert cols == rows and np.array_equal(rp, z["row_ptr"]) and np.array_equal(ci, z["col_idx"])
    assert np.array_equal(v, z["values"])  # %.17g round-trips doubles exactly


def test_csv_precision(tmp_path):
    p = tmp_path / "t.csv"
    io.write_csv(p, ["h", "error"], [[0.1, 1 / 3]])
    a, b = p.read_text().splitlines()[1].split(",")
    assert a == "0.10000000000000001" and float(b) == 1 / 3
