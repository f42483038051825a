"""GPU vs the committed reference fixtures (tests/golden, produced by the
compiled reference, see make_golden.py): the device path reproduces the
reference's own outputs without any CPU checker on the GPU box."""
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2205_03354_b200.cahn_hilliard import CahnHilliardExplicit, CahnHilliardParams, CahnHilliardState, free_energy  # noqa: E402,E501
from paper_2205_03354_b200.grid import BoundaryKind, GridSpec, apply, assemble, composed_apply  # noqa: E402
from paper_2205_03354_b200.linalg import SolveOptions, cg_solve  # noqa: E402
from paper_2205_03354_b200.stencil import bilaplacian, laplacian  # noqa: E402

GOLD = Path(__file__).resolve().parent / "golden"
CSR = sorted(GOLD.glob("csr_*.npz"))


def case(path):
    z = np.load(path)
    dim, acc, kind, n, bc = (int(v) for v in z["meta"])
    g = GridSpec(dim, [n] * dim, float(z["h"]), [0.0] * dim, [BoundaryKind(bc)] * dim)
    s = laplacian(dim, acc) if kind == 1 else bilaplacian(dim, acc)
    return z, s, g


@pytest.mark.parametrize("path", CSR, ids=lambda p: p.stem)
@pytest.mark.parametrize("bits", [64, 32])
def test_gpu_assembly_and_spmv_equal_reference(path, bits):
    z, s, g = case(path)
    m = assemble(s, g, index_bits=bits)
    rp, ci, v = m.to_host()
    assert np.array_equal(rp, z["row_ptr"])
    assert np.array_equal(ci, z["col_idx"])
    assert np.array_equal(v, z["values"])
    # SpMV: same per-row order and rounding as kernels::serial::csr_matvec
    assert np.array_equal(apply(m, z["x"]), z["y"])


@pytest.mark.parametrize("path", CSR, ids=lambda p: p.stem)
def test_gpu_matrix_free_apply_vs_reference(path):
    z, s, g = case(path)
    v = composed_apply(s, g, z["x"])
    y = z["y"]
    assert np.abs(v - y).max() <= 1e-12 * np.abs(y).max()


def test_gpu_cg_vs_reference():
    z, s, g = case(GOLD / "csr_bilap2d_cl17.npz")
    m = assemble(s, g)
    x = cg_solve(m, z["cg_b"], SolveOptions(rel_tol=1e-9))
    assert np.linalg.norm(x - z["cg_x"]) <= 1e-8 * np.linalg.norm(z["cg_x"])


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("formulation", ["factored", "composed"])
def test_gpu_cahn_hilliard_vs_reference(dim, formulation):
    z = np.load(GOLD / f"ch_{dim}d.npz")
    d, n, steps, _ = (int(v) for v in z["meta"])
    kappa, mob, rho, ca, cb = (float(v) for v in z["params"])
    p = CahnHilliardParams(kappa, mob, rho, ca, cb, formulation)
    g = GridSpec(d, [n] * d, float(z["h"]), [0.0] * d, [BoundaryKind.periodic] * d)
    st = CahnHilliardState(g, z["c0"].copy())
    CahnHilliardExplicit(g, p).step(st, float(z["dt"]), steps)
    assert np.linalg.norm(st.c - z["c"]) <= 1e-9 * np.linalg.norm(z["c"])
    assert abs(free_energy(st, p) - float(z["energy"])) <= 1e-12 * abs(float(z["energy"]))
    assert abs(free_energy(z["c0"], p, g) - float(z["energy0"])) <= 1e-12 * abs(float(z["energy0"]))
