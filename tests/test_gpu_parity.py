"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bars (BASELINE.json north_star): CSR row_ptr / col_idx bit-exact (values
too); operator apply <= 1e-12 relative max error; CH fields after N steps
<= 1e-9 relative L2; CG solutions <= 1e-8 relative. Inputs are seeded
(std::mt19937_64 + uniform_real_distribution, the reference's generator).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from paper_2205_03354_b200 import kernels as K  # noqa: E402
from paper_2205_03354_b200.cahn_hilliard import (CahnHilliardExplicit, CahnHilliardParams,  # noqa: E402
                                                 CahnHilliardState, free_energy)
from paper_2205_03354_b200.device import DeviceArray  # noqa: E402
from paper_2205_03354_b200.errors import Errc, StencilkitError  # noqa: E402
from paper_2205_03354_b200.grid import (BoundaryKind, CsrMatrix, DeviceStencil, GridSpec, apply,  # noqa: E402
                                        assemble, composed_apply, composed_apply_repeat, make_grid,
                                        make_periodic_grid)
from paper_2205_03354_b200.linalg import SolveOptions, SolveReport, cg_solve  # noqa: E402
from paper_2205_03354_b200.stencil import (Stencil, StencilSpec, bilaplacian, compose, laplacian,  # noqa: E402
                                           make, scale)


def uniform(seed, n, lo=-1.0, hi=1.0):
    from paper_2205_03354_b200._lib import load

    out = np.empty(n)
    load().sk_fill_uniform_host(seed, n, lo, hi, out.ctypes.data)
    return out


def rel_max(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


# ---------------------------------------------------------------- apply ----
@pytest.mark.parametrize("n", [1024, 256, 100, 37, 130])
def test_apply_2d_13pt_vs_oracle(orc, n):
    g = make_periodic_grid(2, n, 1.0 / n)
    s = bilaplacian(2)
    u = uniform(99, g.unknown_count())
    v = composed_apply(s, g, u)
    assert rel_max(v, orc.apply_direct(s, g, u)) <= 1e-12
    rp, ci, vals = orc.assemble(s, g)
    assert rel_max(v, orc.csr_matvec(rp, ci, vals, u)) <= 1e-12


def test_config1_apply_and_analytic(orc):
    """BASELINE config 1: 1024^2, u = sin(2 pi x) sin(2 pi y) + 1e-3 U(-1,1) (seed 0)."""
    n = 1024
    h = 1.0 / n
    g = make_periodic_grid(2, n, h)
    s = bilaplacian(2)
    x = np.arange(n) * h
    smooth = np.outer(np.sin(2 * np.pi * x), np.sin(2 * np.pi * x)).ravel()  # row j (y), col i (x)
    u = smooth + 1e-3 * uniform(0, n * n)
    v = composed_apply(s, g, u)
    rp, ci, vals = orc.assemble(s, g)
    assert rel_max(v, orc.csr_matvec(rp, ci, vals, u)) <= 1e-12
    # analytic: Delta^2 (sin sin) = 64 pi^4 sin sin, O(h^2) discretisation error (~7.1e-6)
    v0 = composed_apply(s, g, smooth)
    exact = 64 * np.pi ** 4 * smooth
    err = float(np.abs(v0 - exact).max() / np.abs(exact).max())
    assert err <= 1e-5


def test_apply_repeat_graph_matches_single(orc):
    n = 512
    g = make_periodic_grid(2, n, 1.0 / n)
    s = DeviceStencil(bilaplacian(2))
    u = DeviceArray.from_host(uniform(1, n * n))
    v0, v1 = DeviceArray(n * n), DeviceArray(n * n)
    composed_apply_repeat(s, g, u, v0, v1, 7)
    composed_apply_repeat(s, g, u, v0, v1, 7)  # cached graph replay
    single = composed_apply(s, g, u.to_host())
    assert np.array_equal(v0.to_host(), single)
    assert np.array_equal(v1.to_host(), single)


@pytest.mark.parametrize("n", [64, 37, 256])
def test_apply_3d_25pt_vs_oracle(orc, n):
    g = make_periodic_grid(3, n, 1.0 / n)
    s = bilaplacian(3)
    assert DeviceStencil(s).kernel_class == 2
    u = uniform(5, g.unknown_count())
    v = composed_apply(s, g, u)
    assert rel_max(v, orc.apply_direct(s, g, u)) <= 1e-12


@pytest.mark.parametrize("n", [48, 30, 128])
def test_apply_3d_73pt_vs_oracle(orc, n):
    g = make_periodic_grid(3, n, 1.0 / n)
    s = bilaplacian(3, 4)
    assert len(s.entries) == 73 and DeviceStencil(s).kernel_class == 3
    u = uniform(6, g.unknown_count())
    v = composed_apply(s, g, u)
    assert rel_max(v, orc.apply_direct(s, g, u)) <= 1e-12


@pytest.mark.parametrize("bc", [BoundaryKind.periodic, BoundaryKind.simply_supported, BoundaryKind.clamped])
def test_apply_generic_paths(orc, bc):
    # non-symmetric 2D stencil (generic kernel) and the symmetric ones on non-periodic grids
    d1 = make(StencilSpec(1, 2))
    d2 = make(StencilSpec(2, 2))
    from paper_2205_03354_b200.stencil import outer_product

    mixed = outer_product(compose(d1, d2), d2)  # f_(3,2), not symmetric
    for s, dim, n in [(mixed, 2, 29), (bilaplacian(2), 2, 40), (bilaplacian(3), 3, 14), (bilaplacian(3, 4), 3, 15),
                      (compose(d2, d2), 1, 50)]:
        g = make_grid(dim, n, 1.0 / (n - 1), bc)
        u = uniform(7, g.unknown_count())
        v = composed_apply(s, g, u)
        rp, ci, vals = orc.assemble(s, g)
        assert rel_max(v, orc.csr_matvec(rp, ci, vals, u)) <= 1e-12, (dim, n)


# ------------------------------------------------------------ Cahn-Hilliard --
@pytest.mark.parametrize("n,steps", [(128, 50), (100, 20), (256, 10)])
def test_ch_2d_vs_oracle(orc, n, steps):
    p = CahnHilliardParams.from_epsilon(0.01)
    h = 1.0 / n
    dt = 0.25 * h ** 4 / (64 * p.kappa)
    g = make_periodic_grid(2, n, h)
    c0 = 0.05 * uniform(1, g.unknown_count())
    st = CahnHilliardState(g, c0.copy())
    CahnHilliardExplicit(g, p).step(st, dt, steps)
    ref = orc.ch_explicit(2, n, h, p, dt, steps, c0)
    assert np.linalg.norm(st.c - ref) / np.linalg.norm(ref) <= 1e-9
    e_gpu = free_energy(st, p)
    e_ref = orc.free_energy(2, n, h, p, ref)
    assert abs(e_gpu - e_ref) <= 1e-12 * abs(e_ref)


@pytest.mark.parametrize("formulation", ["factored", "composed"])
@pytest.mark.parametrize("n,steps", [(32, 20), (70, 5), (64, 12), (96, 7)])
def test_ch_3d_vs_oracle(orc, n, steps, formulation):
    p = CahnHilliardParams.from_epsilon(0.02, formulation)
    h = 1.0 / n
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    g = make_periodic_grid(3, n, h)
    c0 = 0.05 * uniform(2, g.unknown_count())
    st = CahnHilliardState(g, c0.copy())
    CahnHilliardExplicit(g, p).step(st, dt, steps)
    ref = orc.ch_explicit(3, n, h, p, dt, steps, c0)
    assert np.linalg.norm(st.c - ref) / np.linalg.norm(ref) <= 1e-9
    assert abs(free_energy(st, p) - orc.free_energy(3, n, h, p, ref)) <= 1e-12 * abs(orc.free_energy(3, n, h, p, ref))


def test_ch_graph_chunks_and_remainder(orc):
    # 230 steps = 2 graph replays of 100 + 30 direct launches
    n = 64
    p = CahnHilliardParams.from_epsilon(0.01)
    h = 1.0 / n
    dt = 0.25 * h ** 4 / (64 * p.kappa)
    g = make_periodic_grid(2, n, h)
    c0 = 0.05 * uniform(3, g.unknown_count())
    st = CahnHilliardState(g, c0.copy())
    CahnHilliardExplicit(g, p).step(st, dt, 230)
    ref = orc.ch_explicit(2, n, h, p, dt, 230, c0)
    assert np.linalg.norm(st.c - ref) / np.linalg.norm(ref) <= 1e-9


@pytest.mark.parametrize("n,steps", [(64, 230), (128, 100)])
def test_ch_3d_padded_path(orc, n, steps, sk_option):
    # >= 100 steps of the 3D factored form run as graph chunks through ghost-padded
    # fields (TMA kernel); the result is bit-identical to the plain cp.async path
    # and matches the oracle
    p = CahnHilliardParams.from_epsilon(0.02)
    h = 1.0 / n
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    g = make_periodic_grid(3, n, h)
    c0 = 0.05 * uniform(4, g.unknown_count())
    out = {}
    for flag in ("1", "0"):
        sk_option("ch_padded", int(flag))
        st = CahnHilliardState(g, c0.copy())
        CahnHilliardExplicit(g, p).step(st, dt, steps)
        out[flag] = st.c.copy()
    assert np.array_equal(out["1"], out["0"])
    ref = orc.ch_explicit(3, n, h, p, dt, steps, c0)
    assert np.linalg.norm(out["1"] - ref) / np.linalg.norm(ref) <= 1e-9


@pytest.mark.parametrize("steps", [1, 2, 3, 20, 101, 102, 203])
def test_ch_3d_chunking_any_step_count(orc, steps, sk_option):
    # every step count >= 2 runs as chunk graphs (padded TMA path for the 3D
    # factored form): bit-identical to the plain path, the result in the buffer
    # the ping-pong parity names, and within the bar of the oracle
    n = 64
    p = CahnHilliardParams.from_epsilon(0.02)
    h = 1.0 / n
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    g = make_periodic_grid(3, n, h)
    c0 = 0.05 * uniform(8, g.unknown_count())
    out = {}
    for flag in (1, 0):
        sk_option("ch_padded", flag)
        st = CahnHilliardExplicit(g, p)
        c, s = DeviceArray.from_host(c0), DeviceArray(g.unknown_count())
        res = st.run_device(c, s, dt, steps)
        assert (res is s) == bool(steps % 2)
        out[flag] = res.to_host()
    assert np.array_equal(out[1], out[0])
    ref = orc.ch_explicit(3, n, h, p, dt, steps, c0)
    assert np.linalg.norm(out[1] - ref) / np.linalg.norm(ref) <= 1e-9


def test_ch_3d_concurrent_streams(lib):
    # two steppers of the same grid size on two streams, issued back to back
    # without a sync: each stream has its own ghost-padded pair, so the runs
    # cannot corrupt each other; results equal the sequential runs
    import ctypes as C

    n, steps = 64, 100
    p = CahnHilliardParams.from_epsilon(0.02)
    h = 1.0 / n
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    g = make_periodic_grid(3, n, h)
    fields = [0.05 * uniform(20 + k, g.unknown_count()) for k in range(2)]
    seq = []
    for f in fields:
        st = CahnHilliardState(g, f.copy())
        CahnHilliardExplicit(g, p).step(st, dt, steps)
        seq.append(st.c)
    streams = [C.c_void_p(), C.c_void_p()]
    for s_ in streams:
        assert lib.sk_stream_create(C.byref(s_)) == 0
    try:
        steppers = [CahnHilliardExplicit(g, p) for _ in fields]
        bufs = [(DeviceArray.from_host(f), DeviceArray(g.unknown_count())) for f in fields]
        for rep in range(3):  # replays of the cached graphs interleave too
            for k in range(2):
                bufs[k][0].upload(fields[k])
            res = [steppers[k].run_device(bufs[k][0], bufs[k][1], dt, steps, streams[k]) for k in range(2)]
            for s_ in streams:
                assert lib.sk_stream_sync(s_) == 0
            for k in range(2):
                assert np.array_equal(res[k].to_host(), seq[k]), (rep, k)
    finally:
        for s_ in streams:
            lib.sk_stream_destroy(s_)


def test_ch_rejects_unknown_formulation():
    g = make_periodic_grid(3, 32, 1.0 / 32)
    p = CahnHilliardParams.from_epsilon(0.02)
    st = CahnHilliardExplicit(g, p)
    st._p.formulation = 2
    c, s = DeviceArray(g.unknown_count()), DeviceArray(g.unknown_count())
    with pytest.raises(StencilkitError) as e:
        st.run_device(c, s, 1e-9, 3)
    assert e.value.code == Errc.invalid_argument


def test_ch_rejects_non_periodic():
    g = make_grid(2, 32, 1.0 / 31, BoundaryKind.clamped)
    with pytest.raises(StencilkitError) as e:
        CahnHilliardExplicit(g, CahnHilliardParams())
    assert e.value.code == Errc.non_periodic


# ---------------------------------------------------------------- assembly --
CASES = [
    (2, 2, 37, BoundaryKind.periodic), (2, 2, 64, BoundaryKind.simply_supported), (2, 2, 65, BoundaryKind.clamped),
    (2, 2, 5, BoundaryKind.periodic), (2, 2, 5, BoundaryKind.clamped), (3, 2, 17, BoundaryKind.periodic),
    (3, 2, 18, BoundaryKind.clamped), (3, 4, 21, BoundaryKind.clamped), (3, 4, 9, BoundaryKind.periodic),
    (3, 4, 11, BoundaryKind.simply_supported), (3, 4, 10, BoundaryKind.clamped),
]


@pytest.mark.parametrize("dim,acc,n,bc", CASES)
@pytest.mark.parametrize("bits", [64, 32])
def test_assembly_bit_exact(orc, dim, acc, n, bc, bits):
    s = bilaplacian(dim, acc)
    g = make_grid(dim, n, 1.0 / (n if bc == BoundaryKind.periodic else n - 1), bc)
    m = assemble(s, g, index_bits=bits)
    rp, ci, v = m.to_host()
    orp, oci, ov = orc.assemble(s, g)
    assert np.array_equal(rp, orp)
    assert np.array_equal(ci, oci)
    assert np.array_equal(v, ov)  # values too: same sort + merge order


def test_assembly_laplacians_and_identity(orc):
    for s, dim in [(laplacian(2, 2), 2), (laplacian(3, 2), 3), (laplacian(3, 4), 3), (Stencil.identity(2), 2)]:
        for bc in BoundaryKind:
            g = make_grid(dim, 12, 0.25, bc)
            m = assemble(s, g)
            got = m.to_host()
            want = orc.assemble(s, g)
            assert all(np.array_equal(a, b) for a, b in zip(got, want))


def test_assembly_large_sampled_rows(orc):
    """cfg5-like 73-point clamped at 129^3 (127^3 rows): sampled rows vs the oracle's row algorithm."""
    s = bilaplacian(3, 4)
    n = 129
    g = make_grid(3, n, 1.0 / (n - 1), BoundaryKind.clamped)
    m = assemble(s, g)
    rp, ci, v = m.to_host()
    rows = m.rows
    assert rows == 127 ** 3
    rng = np.random.default_rng(4)
    sample = list(rng.integers(0, rows, 3000)) + list(range(0, 2000)) + list(range(rows - 2000, rows))
    for r in sample:
        cols, vals = orc.assemble_row(s, g, int(r))
        assert np.array_equal(ci[rp[r]:rp[r + 1]], cols)
        assert np.array_equal(v[rp[r]:rp[r + 1]], vals)
    assert np.all(np.diff(rp) > 0)


@pytest.mark.parametrize("bits", [64, 32])
def test_assemble_into_reuses_the_matrix(orc, bits):
    # re-assembly into an existing matrix (new h -> new weights, same pattern)
    # is bit-identical to a fresh assembly; the cached SELL copy / CG plan of
    # the matrix follow the new values; a shape change is rejected
    from paper_2205_03354_b200.grid import assemble_into

    s = bilaplacian(3, 4)
    g1 = make_grid(3, 21, 1.0 / 20, BoundaryKind.clamped)
    g2 = make_grid(3, 21, 1.0 / 7, BoundaryKind.clamped)
    m = assemble(s, g1, index_bits=bits)
    x = uniform(5, m.rows)
    y1 = apply(m, x)  # builds the SELL copy
    assemble_into(s, g2, m)
    rp, ci, v = m.to_host()
    orp, oci, ov = orc.assemble(s, g2)
    assert np.array_equal(rp, orp) and np.array_equal(ci, oci) and np.array_equal(v, ov)
    y2 = apply(m, x)
    assert np.array_equal(y2, apply(assemble(s, g2, index_bits=bits), x))
    assert not np.array_equal(y1, y2)
    with pytest.raises(StencilkitError) as e:
        assemble_into(s, make_grid(3, 19, 1.0 / 18, BoundaryKind.clamped), m)
    assert e.value.code == Errc.shape_mismatch


def test_assembly_errors():
    with pytest.raises(StencilkitError) as e:
        assemble(bilaplacian(2), make_periodic_grid(2, 4, 1.0))
    assert e.value.code == Errc.stencil_wider_than_grid
    with pytest.raises(StencilkitError) as e:
        assemble(bilaplacian(2), make_periodic_grid(3, 8, 1.0))
    assert e.value.code == Errc.dim_mismatch


# ------------------------------------------------------------ SpMV + BLAS --
def test_spmv_bit_exact_vs_serial(orc, ref):
    """test_kernels.cpp:26-35: periodic bilap on 37^2, x ~ mt19937_64(99)."""
    g = make_periodic_grid(2, 37, 1.0)
    s = bilaplacian(2)
    m = assemble(s, g)
    x = uniform(99, m.rows)
    rp, ci, v = orc.assemble(s, g)
    assert np.array_equal(apply(m, x), orc.csr_matvec(rp, ci, v, x))


@pytest.mark.parametrize("bits", [64, 32])
def test_spmv_bit_exact_large(orc, bits):
    s = bilaplacian(3, 4)
    g = make_grid(3, 66, 1.0 / 65, BoundaryKind.clamped)
    m = assemble(s, g, index_bits=bits)
    x = uniform(11, m.rows)
    rp, ci, v = orc.assemble(s, g)
    assert np.array_equal(apply(m, x), orc.csr_matvec(rp, ci, v, x))


def test_blas(orc):
    """test_kernels.cpp:37-60 on the device."""
    x = uniform(7, 10001)
    y = uniform(8, 10001)
    dx, dy = DeviceArray.from_host(x), DeviceArray.from_host(y)
    K.axpy(0.37, dx, dy)
    y2 = orc.axpy(0.37, x, y)
    assert np.array_equal(dy.to_host(), y2)
    K.xpby(dx, -1.25, dy)
    y3 = orc.xpby(x, -1.25, y2)
    assert np.array_equal(dy.to_host(), y3)
    a = uniform(13, 50000)
    b = uniform(14, 50000)
    assert K.dot(a, b) == pytest.approx(orc.dot(a, b), rel=1e-13)
    assert K.sum(a) == pytest.approx(orc.sum(a), rel=1e-12)
    assert K.nrm2(a) == pytest.approx(orc.nrm2(a), rel=1e-13)
    assert K.minmax(a) == orc.minmax(a)
    big = uniform(15, 5_000_001)
    assert K.sum(big) == pytest.approx(orc.sum(big), rel=1e-10)


# ---------------------------------------------------------------------- CG --
def test_cg_identity():
    g = make_periodic_grid(1, 32, 1.0)
    m = assemble(Stencil.identity(1), g)
    b = uniform(3, 32, -2, 2)
    assert np.allclose(cg_solve(m, b), b, rtol=1e-12, atol=0)


def test_cg_poisson_periodic_deflated():
    """test_linalg.cpp:28-59: -d2 on a sine mode, mean-free, true residual <= 1e-12 ||b||."""
    n = 64
    h = 1.0 / n
    g = make_periodic_grid(1, n, h)
    d2 = make(StencilSpec(2, 2))
    m = assemble(scale(d2, -1), g)
    theta = 2 * np.pi * 3 / n
    lam = (2 - 2 * np.cos(theta)) / (h * h)
    b = np.sin(theta * np.arange(n))
    x = cg_solve(m, b, SolveOptions(rel_tol=1e-12, deflate_mean=True))
    assert abs(x.sum()) <= 1e-12 * n
    assert np.allclose(x, b / lam, rtol=1e-9, atol=1e-15)
    r = np.linalg.norm(b - apply(m, x))
    assert r <= 1e-12 * np.linalg.norm(b)


def test_cg_failures():
    g = make_periodic_grid(1, 16, 1.0)
    b = np.zeros(16)
    b[3], b[7] = 1.0, -1.0
    with pytest.raises(StencilkitError) as e:
        cg_solve(assemble(make(StencilSpec(2, 2)), g), b)
    assert e.value.code == Errc.no_convergence
    with pytest.raises(StencilkitError) as e:
        cg_solve(assemble(scale(make(StencilSpec(2, 2)), -1), g), b, SolveOptions(rel_tol=1e-14, max_iter=2))
    assert e.value.code == Errc.no_convergence


@pytest.mark.parametrize("dim,acc,intervals,tol", [(2, 2, 32, 1e-10), (2, 2, 64, 1e-10), (3, 4, 16, 1e-10)])
def test_cg_biharmonic_clamped_vs_oracle(orc, dim, acc, intervals, tol):
    s = bilaplacian(dim, acc)
    g = make_grid(dim, intervals + 1, 1.0 / intervals, BoundaryKind.clamped)
    m = assemble(s, g)
    f, u = orc.biharmonic_clamped(dim, intervals)
    rep = SolveReport()
    x = cg_solve(m, f, SolveOptions(rel_tol=tol), rep)
    rp, ci, v = orc.assemble(s, g)
    xo, status, iters, _ = orc.cg_solve(rp, ci, v, f, tol)
    assert status == 0
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) <= 1e-8
    assert rep.true_rel_residual <= tol
    assert abs(rep.iterations - iters) <= max(5, iters // 20)


@pytest.mark.parametrize("dims,steps", [((64, 32, 5), 100), ((128, 64, 6), 230), ((96, 40, 7), 120), ((64, 32, 9), 100),
                                        ((128, 48), 150), ((67, 36, 9), 60), ((130, 34, 8), 40)])
def test_ch_noncubic_grids(orc, dims, steps, sk_option):
    # non-cubic periodic grids, tiny z extents (z wrap inside one chunk), the
    # ghost-padded TMA path (whole tiles) and the plain path, vs the oracle
    from paper_2205_03354_b200.grid import GridSpec

    dim = len(dims)
    p = CahnHilliardParams.from_epsilon(0.02)
    h = 1.0 / max(dims)
    dt = 0.2 * h ** 4 / (144 * p.kappa)
    g = GridSpec(dim=dim, n=list(dims), h=h, origin=[0.0] * dim, bc=[BoundaryKind.periodic] * dim)
    c0 = 0.05 * uniform(6, g.unknown_count())
    out = {}
    for flag in ("1", "0"):
        sk_option("ch_padded", int(flag))
        st = CahnHilliardState(g, c0.copy())
        CahnHilliardExplicit(g, p).step(st, dt, steps)
        out[flag] = st.c.copy()
    assert np.array_equal(out["1"], out["0"])
    ref = orc.ch_explicit_dims(dims, h, p, dt, steps, c0)
    assert np.linalg.norm(out["1"] - ref) / np.linalg.norm(ref) <= 1e-9


def test_ch_rejects_narrow_axes():
    # the 25-point B needs 5 points per periodic axis (grid.cpp:66-75), and every
    # grid at least 3 points per axis (grid.cpp:17-25)
    from paper_2205_03354_b200.grid import GridSpec

    p = CahnHilliardParams.from_epsilon(0.02)
    for dims, code in [((64, 32, 4), Errc.stencil_wider_than_grid), ((64, 32, 2), Errc.invalid_argument)]:
        g = GridSpec(dim=3, n=list(dims), h=0.1, origin=[0.0] * 3, bc=[BoundaryKind.periodic] * 3)
        with pytest.raises(StencilkitError) as e:
            st = CahnHilliardState(g, np.zeros(int(np.prod(dims))))
            CahnHilliardExplicit(g, p).step(st, 1e-9, 1)
        assert e.value.code == code
