"""CPU: pin the plain-C oracle (oracle/sk_oracle.c) and the host stencil algebra.

Against (a) the golden fixtures generated from the compiled reference
(tests/golden/make_golden.py), (b) the reference's own known-answer tests
(weights of test_generators.cpp:12-26,54-75; sparsity of test_grid.cpp:60-95),
and (c) when the compiled reference is present here, live comparisons on
random stencils and grids. Assembly, csr_matvec, the CH restatement, the
serial free energy and the generator are bit-exact; CG is bit-exact with the
single-threaded reference.
"""
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

from paper_2205_03354_b200.errors import Errc, StencilkitError
from paper_2205_03354_b200.grid import BoundaryKind, GridSpec, make_grid, make_periodic_grid
from paper_2205_03354_b200.stencil import (Stencil, StencilSpec, bilaplacian, compose, from_entries, laplacian,
                                           make, outer_product, scale, to_double, weight_sum)

GOLD = Path(__file__).resolve().parent / "golden"


def stencil_from_fixture(z, key):
    off, num, den, hp = z[key + "_off"], z[key + "_num"], z[key + "_den"], int(z[key + "_hp"])
    return from_entries(off.shape[1], hp, [(tuple(o), Fraction(int(n), int(d))) for o, n, d in zip(off, num, den)])


def grid_for(meta, h):
    dim, acc, kind, n, bc = (int(v) for v in meta)
    return GridSpec(dim, [n] * dim, float(h), [0.0] * dim, [BoundaryKind(bc)] * dim)


def stencil_for(meta):
    dim, acc, kind = (int(v) for v in meta[:3])
    return laplacian(dim, acc) if kind == 1 else bilaplacian(dim, acc)


# ------------------------------------------------------------ stencil host --
def test_generators_known_answers():
    """test_generators.cpp:12-26 (exact 1D stencils)."""
    def s1(hp, d):
        return Stencil(1, hp, {(k,): Fraction(v) for k, v in d.items()})

    assert make(StencilSpec(1, 2)) == s1(-1, {1: Fraction(1, 2), -1: Fraction(-1, 2)})
    assert make(StencilSpec(2, 2)) == s1(-2, {1: 1, 0: -2, -1: 1})
    assert make(StencilSpec(1, 4)) == s1(-1, {1: Fraction(8, 12), 2: Fraction(-1, 12), -2: Fraction(1, 12),
                                              -1: Fraction(-8, 12)})
    assert make(StencilSpec(2, 1, "forward")) == s1(-2, {2: 1, 1: -2, 0: 1})
    assert make(StencilSpec(1, 2, "forward")) == s1(-1, {0: Fraction(-3, 2), 1: 2, 2: Fraction(-1, 2)})
    assert make(StencilSpec(1, 1, "forward")) == s1(-1, {1: 1, 0: -1})
    # centred stencils round odd accuracy up (test_generators.cpp:47-50)
    assert make(StencilSpec(1, 1)) == make(StencilSpec(1, 2))


def test_laplacian_and_bilaplacian_weights():
    """test_generators.cpp:54-75: 5-point cross, 7-point (centre -6), 13-point biharmonic."""
    assert laplacian(1, 2) == make(StencilSpec(2, 2))
    five = {(0, 1): 1, (0, -1): 1, (1, 0): 1, (-1, 0): 1, (0, 0): -4}
    assert laplacian(2, 2) == Stencil(2, -2, {k: Fraction(v) for k, v in five.items()})
    lap3 = laplacian(3, 2)
    assert len(lap3.entries) == 7 and lap3.entries[(0, 0, 0)] == -6
    b = bilaplacian(2)
    assert len(b.entries) == 13
    assert b.entries[(0, 0)] == 20 and b.entries[(0, 1)] == -8 and b.entries[(1, -1)] == 2 and b.entries[(0, -2)] == 1
    with pytest.raises(StencilkitError) as e:
        laplacian(2, 3)
    assert e.value.code == Errc.unsupported_accuracy
    with pytest.raises(StencilkitError):
        laplacian(4, 2)


def test_composed_stencils_match_reference_fixture():
    z = np.load(GOLD / "stencils.npz")
    for dim, acc in [(1, 2), (2, 2), (3, 2), (1, 4), (3, 4)]:
        for name, s in [("lap", laplacian(dim, acc)), ("bilap", bilaplacian(dim, acc))]:
            key = f"st_{name}{dim}d_a{acc}"
            ref = stencil_from_fixture(z, key)
            assert s == ref, key
            offs, coeffs = s.flat()
            assert np.array_equal(np.array(offs).reshape(-1, dim), z[key + "_off"])
            assert np.array_equal(np.array(coeffs), z[key + "_coeff"])  # truncating to_double
    b73 = bilaplacian(3, 4)
    assert len(b73.entries) == 73 and weight_sum(b73) == 0
    assert b73.entries[(0, 0, 0)] == Fraction(1607, 24) and b73.entries[(4, 0, 0)] == Fraction(1, 144)


def test_to_double_truncates():
    """mpq_get_d semantics behind Rational::to_double (rational.hpp:32)."""
    for q in [Fraction(1, 3), Fraction(-2, 3), Fraction(1607, 24), Fraction(-182, 9), Fraction(1, 144), Fraction(7)]:
        d = to_double(q)
        assert abs(Fraction(d)) <= abs(q)
        assert abs(q - Fraction(d)) < abs(Fraction(np.nextafter(d, np.inf if q > 0 else -np.inf)) - Fraction(d))


def test_stencil_algebra_errors():
    with pytest.raises(StencilkitError) as e:
        Stencil(2, 0, {(0, 0): Fraction(0)})
    assert e.value.code == Errc.empty_stencil
    with pytest.raises(StencilkitError) as e:
        scale(laplacian(2, 2), 0)
    assert e.value.code == Errc.zero_scale
    with pytest.raises(StencilkitError) as e:
        compose(laplacian(2, 2), laplacian(3, 2))
    assert e.value.code == Errc.dim_mismatch
    # outer product of 1D stencils = 2D mixed derivative (experiments.cpp:75-78 pattern)
    m = outer_product(make(StencilSpec(1, 2)), make(StencilSpec(1, 2)))
    assert m.dim == 2 and m.h_power == -2 and len(m.entries) == 4


def test_grid_validation():
    """test_grid.cpp:200-212."""
    g = GridSpec(2, [4], 1.0, [0.0, 0.0], [BoundaryKind.periodic] * 2)
    with pytest.raises(StencilkitError):
        g.validate()
    with pytest.raises(StencilkitError):
        make_periodic_grid(1, 2, 1.0)
    assert make_grid(2, 17, 1 / 16, BoundaryKind.clamped).unknown_count() == 15 * 15


# ------------------------------------------------------------ C oracle -----
@pytest.mark.parametrize("path", sorted(GOLD.glob("csr_*.npz")), ids=lambda p: p.stem)
def test_oracle_assembly_and_matvec_bit_exact(orc, path):
    z = np.load(path)
    s = stencil_for(z["meta"])
    g = grid_for(z["meta"], z["h"])
    rp, ci, v = orc.assemble(s, g)
    assert np.array_equal(rp, z["row_ptr"]) and np.array_equal(ci, z["col_idx"]) and np.array_equal(v, z["values"])
    assert np.array_equal(orc.csr_matvec(rp, ci, v, z["x"]), z["y"])
    # row-at-a-time restatement (used for sampled checks at config sizes)
    for r in [0, 1, len(rp) // 2, len(rp) - 2]:
        cols, vals = orc.assemble_row(s, g, r)
        assert np.array_equal(cols, ci[rp[r]:rp[r + 1]]) and np.array_equal(vals, v[rp[r]:rp[r + 1]])
    if "cg_x" in z.files:
        x, st, it, tr = orc.cg_solve(rp, ci, v, z["cg_b"], 1e-9)
        assert st == int(z["cg_status"]) == 0
        assert np.array_equal(x, z["cg_x"])  # single-threaded reference: same reduction order


def test_sparsity_known_answers(orc):
    """test_grid.cpp:60-95: 5N / 13N entries on periodic grids, exact fill percentages."""
    lap, bil = laplacian(2, 2), bilaplacian(2)
    for h, size, lp, bp in [(8.0, 625, 0.8, 2.08), (4.0, 2500, 0.2, 0.52), (2.0, 10000, 0.05, 0.13)]:
        g = make_periodic_grid(2, int(200 / h), h)
        _, _, vl = orc.assemble(lap, g)
        _, _, vb = orc.assemble(bil, g)
        assert g.unknown_count() == size and vl.size == 5 * size and vb.size == 13 * size
        assert 100.0 * vl.size / (size * size) == lp and 100.0 * vb.size / (size * size) == bp


@pytest.mark.parametrize("dim", [2, 3])
def test_oracle_cahn_hilliard_bit_exact(orc, dim):
    z = np.load(GOLD / f"ch_{dim}d.npz")
    d, n, steps, _ = (int(v) for v in z["meta"])

    class P:
        kappa, mobility, rho_w, c_alpha, c_beta = (float(v) for v in z["params"])

    c = orc.ch_explicit(d, n, float(z["h"]), P, float(z["dt"]), steps, z["c0"])
    assert np.array_equal(c, z["c"])
    assert orc.free_energy(d, n, float(z["h"]), P, z["c0"]) == float(z["energy0"])
    assert orc.free_energy(d, n, float(z["h"]), P, c) == float(z["energy"])


def test_oracle_generator_and_fit(orc):
    z = np.load(GOLD / "uniform.npz")
    for s in (0, 1, 2, 3, 99):
        assert np.array_equal(orc.uniform(s, 2000), z[f"seed{s}"])
    # fit_loglog on an exact power law recovers slope and coefficient
    hs = [2.0 ** -k for k in range(2, 7)]
    slope, coeff, resid = orc.fit_loglog(hs, [3.0 * h ** 2 for h in hs])
    assert abs(slope - 2.0) < 1e-12 and abs(coeff - 3.0) < 1e-10 and resid < 1e-12
    with pytest.raises(ValueError):
        orc.fit_loglog(hs[:2], [1.0, 2.0])


def test_oracle_blas_serial_semantics(orc):
    rng = np.random.default_rng(7)
    x, y = rng.uniform(-1, 1, 1001), rng.uniform(-1, 1, 1001)
    assert np.array_equal(orc.axpy(0.37, x, y), y + 0.37 * x)
    assert np.array_equal(orc.xpby(x, -1.25, y), x + (-1.25) * y)
    acc = 0.0
    for a, b in zip(x, y):
        acc += a * b
    assert orc.dot(x, y) == acc
    assert orc.minmax(x) == (x.min(), x.max())


def test_biharmonic_manufactured_rhs(orc):
    """f = Delta^2 u for u = prod sin^2(pi x_i): compare with a symbolic finite check."""
    N = 32
    f, u = orc.biharmonic_clamped(2, N)
    h = 1.0 / N
    x = (np.arange(N - 1) + 1) * h
    a = np.sin(np.pi * x) ** 2
    a2 = 2 * np.pi ** 2 * np.cos(2 * np.pi * x)
    a4 = -8 * np.pi ** 4 * np.cos(2 * np.pi * x)
    want = (np.outer(a, a4) + 2 * np.outer(a2, a2) + np.outer(a4, a)).ravel()
    assert np.allclose(f, want, rtol=1e-13, atol=1e-9)
    assert np.allclose(u, np.outer(a, a).ravel(), rtol=1e-15)


# ---------------------------------------------- live vs compiled reference --
def random_stencil(rng, dim, max_support=3):
    """testutil::random_stencil (test_util.hpp:19-35) analogue."""
    entries = {}
    for _ in range(rng.integers(1, 6)):
        off = tuple(int(v) for v in rng.integers(-max_support, max_support + 1, dim))
        num = int(rng.integers(-6, 7)) or 1
        entries[off] = Fraction(num, int(rng.integers(1, 5)))
    return Stencil(dim, int(rng.integers(-2, 1)), entries)


def test_oracle_vs_reference_random_stencils(orc, ref):
    rng = np.random.default_rng(2024)
    for trial in range(40):
        dim = 1 + trial % 3
        s = random_stencil(rng, dim, 2)
        bc = BoundaryKind(trial % 3)
        n = int(rng.integers(6, 11))
        g = make_grid(dim, n, 0.5, bc)
        offs = np.array([o for o in s.entries]).reshape(-1, dim)
        num = [c.numerator for c in s.entries.values()]
        den = [c.denominator for c in s.entries.values()]
        want = ref.assemble_entries(dim, offs, num, den, s.h_power, [n] * dim, 0.5, [int(bc)] * dim)
        got = orc.assemble(s, g)
        assert all(np.array_equal(a, b) for a, b in zip(got, want)), (trial, s.entries)


def test_oracle_vs_reference_config_sizes(orc, ref):
    """Full-row-count assembly at a config-1 grid (1024^2 periodic) and config-2/5 style clamped grids."""
    for dim, acc, n, bc, h in [(2, 2, 1024, 0, 1 / 1024), (2, 2, 257, 2, 1 / 256), (3, 4, 33, 2, 1 / 32)]:
        s = bilaplacian(dim, acc)
        g = make_grid(dim, n, h, BoundaryKind(bc))
        got = orc.assemble(s, g)
        want = ref.assemble(dim, acc, 2, [n] * dim, h, [bc] * dim)
        assert all(np.array_equal(a, b) for a, b in zip(got, want))


# ------------------------------------------------------------- IMEX (§8f 1) --
@pytest.mark.parametrize("path", sorted(GOLD.glob("imex_*.npz")), ids=lambda p: p.stem)
def test_oracle_imex_bit_exact(orc, path):
    # the C restatement of CahnHilliardStepper::step (order 1, order 2, and the
    # AB2 re-bootstrap on a dt change) reproduces the reference run bit for bit
    from paper_2205_03354_b200.cahn_hilliard import CahnHilliardParams

    d = np.load(path)
    dim, n = (int(x) for x in d["meta"])
    h = float(d["h"])
    assert np.array_equal(orc.ch_init(dim, n, h, 0.5, 0.01), d["c0"])
    seq = [(float(a), int(b), int(c)) for a, b, c in d["seq"]]
    c = orc.ch_imex_seq(dim, n, h, CahnHilliardParams(), seq, d["c0"])
    assert np.array_equal(c, d["c"])


def test_oracle_identity_plus_scaled_vs_reference(orc, ref):
    # linalg.cpp:224-251 on assembled operators, incl. a missing diagonal
    from oracle.ffi import RefCsr

    for dim, acc, n in [(2, 2, 9), (3, 2, 5)]:
        m = RefCsr(ref, dim, acc, 2, [n] * dim, 1.0, [0] * dim)  # bilaplacian, periodic
        rp, ci, v = m.arrays()
        for alpha in (0.37, -1.0 / v[0] if v[0] else 1.0):
            out = ref.L.skref_identity_plus_scaled(m.h, alpha)
            rows, nnz = ref.L.skref_csr_rows(out), ref.L.skref_csr_nnz(out)
            r2, c2, v2 = np.empty(rows + 1, np.int64), np.empty(nnz, np.int64), np.empty(nnz)
            ref.L.skref_csr_copy(out, r2.ctypes.data, c2.ctypes.data, v2.ctypes.data)
            ref.L.skref_csr_free(out)
            r1, c1, v1 = orc.identity_plus_scaled(rp, ci, v, alpha)
            assert np.array_equal(r1, r2) and np.array_equal(c1, c2) and np.array_equal(v1, v2)
    # a matrix without diagonal entries: the reference inserts 1.0 in sorted position
    rp = np.array([0, 2, 3, 4], np.int64)
    ci = np.array([1, 2, 0, 1], np.int64)
    v = np.array([1.0, 2.0, 3.0, 4.0])
    r, c, vals = orc.identity_plus_scaled(rp, ci, v, 0.5)
    assert r.tolist() == [0, 3, 5, 7]
    assert c.tolist() == [0, 1, 2, 0, 1, 1, 2]
    assert vals.tolist() == [1.0, 0.5, 1.0, 1.5, 1.0, 2.0, 1.0]


# --------------------------------------------------------- spectral (§8f 2) --
def test_oracle_spectral_vs_reference(orc, ref):
    # periodic_spectrum eigenvalues / radius / condition and power_iteration
    # (linalg.cpp:74-106,149-193): the C restatement equals the reference
    import ctypes

    from oracle.ffi import RefCsr
    from paper_2205_03354_b200.stencil import bilaplacian, laplacian

    ref.L.skref_set_threads(1)
    for dim, acc, kind, n, h in [(2, 2, 2, (12, 10), 0.5), (3, 2, 2, (6, 5, 7), 1.0), (1, 2, 1, (16,), 0.25),
                                 (2, 4, 2, (9, 9), 1.0)]:
        s = bilaplacian(dim, acc) if kind == 2 else laplacian(dim, acc)
        g = GridSpec(dim=dim, n=list(n), h=h, origin=[0.0] * dim, bc=[BoundaryKind.periodic] * dim)
        for shift, scale in [(0.0, 1.0), (1.0, 0.25)]:
            e_ref, rho_ref, _sym, cond_ref = ref.periodic_spectrum(dim, acc, kind, n, h, shift, scale)
            e, rho, cond = orc.periodic_eigen(s, g, shift, scale)
            assert np.array_equal(e, e_ref) and rho == rho_ref and cond == cond_ref
        m = RefCsr(ref, dim, acc, kind, list(n), h, [0] * dim)
        out = ctypes.c_double()
        assert ref.L.skref_power_iteration(m.h, 1e-8, 20240801, 2_000_000, ctypes.byref(out)) == 0
        lam, its = orc.power_iteration(*m.arrays(), 1e-8)
        assert lam == out.value, (lam, out.value)


def test_oracle_csr_matmul_vs_reference(orc, ref):
    # csr_matmul (linalg.cpp:253-283): the C restatement equals the reference
    from oracle.ffi import RefCsr

    for dim, acc_a, kind_a, acc_b, kind_b, n, bc in [(2, 2, 1, 2, 2, (9, 8), 0), (3, 2, 2, 2, 1, (6, 6, 7), 0),
                                                    (2, 4, 1, 2, 1, (12, 11), 1), (1, 2, 2, 4, 2, (17,), 0)]:
        a = RefCsr(ref, dim, acc_a, kind_a, list(n), 0.5, [bc] * dim)
        b = RefCsr(ref, dim, acc_b, kind_b, list(n), 0.5, [bc] * dim)
        out = ref.L.skref_csr_matmul(b.h, a.h)
        rows, nnz = ref.L.skref_csr_rows(out), ref.L.skref_csr_nnz(out)
        r2, c2, v2 = np.empty(rows + 1, np.int64), np.empty(nnz, np.int64), np.empty(nnz)
        ref.L.skref_csr_copy(out, r2.ctypes.data, c2.ctypes.data, v2.ctypes.data)
        ref.L.skref_csr_free(out)
        r1, c1, v1 = orc.csr_matmul(b.arrays(), a.arrays())
        assert np.array_equal(r1, r2) and np.array_equal(c1, c2) and np.array_equal(v1, v2)
