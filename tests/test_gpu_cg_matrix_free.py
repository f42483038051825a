"""Matrix-free CG (sk_cg_solve_stencil): the composed stencil applied by the
streaming kernels on clamped / simply-supported grids instead of the
assembled CSR. Agrees with the reference-semantics CSR solve (oracle) to the
CG parity bar (1e-8 relative), on the configs' manufactured problems."""
import numpy as np
import pytest

from paper_2205_03354_b200.grid import BoundaryKind, DeviceStencil, assemble, composed_apply, make_grid
from paper_2205_03354_b200.linalg import SolveOptions, SolveReport, cg_solve, cg_solve_stencil
from paper_2205_03354_b200.stencil import bilaplacian

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dim,acc,intervals", [(2, 2, 32), (2, 2, 64), (3, 2, 16), (3, 4, 16)])
def test_matrix_free_cg_vs_oracle(orc, dim, acc, intervals):
    g = make_grid(dim, intervals + 1, 1.0 / intervals, BoundaryKind.clamped)
    s = bilaplacian(dim, acc)
    f, _ = orc.biharmonic_clamped(dim, intervals) if acc == 2 else (np.sin(np.arange(g.unknown_count())), None)
    rp, ci, vals = orc.assemble(s, g)
    xo, status, its_o, _ = orc.cg_solve(rp, ci, vals, f, 1e-10)
    assert status == 0
    rep = SolveReport()
    x = cg_solve_stencil(s, g, f, SolveOptions(rel_tol=1e-10), rep)
    assert np.linalg.norm(x - xo) <= 1e-8 * np.linalg.norm(xo)
    assert rep.true_rel_residual <= 1e-10
    assert abs(rep.iterations - its_o) <= max(3, 0.05 * its_o)


def test_matrix_free_operator_equals_csr_on_every_bc(orc):
    # the streaming kernels' boundary handling reproduces assemble's rows
    for bc in (BoundaryKind.clamped, BoundaryKind.simply_supported, BoundaryKind.periodic):
        for dim, acc, n in [(2, 2, 70), (3, 2, 21), (3, 4, 19)]:
            g = make_grid(dim, n, 1.0 / (n - 1), bc)
            s = bilaplacian(dim, acc)
            u = np.cos(np.arange(g.unknown_count()) * 0.37)
            v = composed_apply(s, g, u)
            rp, ci, vals = orc.assemble(s, g)
            ref = orc.csr_matvec(rp, ci, vals, u)
            assert np.abs(v - ref).max() <= 1e-12 * np.abs(ref).max(), (bc, dim, acc)


def test_matrix_free_and_csr_cg_agree_config2():
    # config 2 at N = 256: the two device solvers reach the same solution
    N = 256
    g = make_grid(2, N + 1, 1.0 / N, BoundaryKind.clamped)
    s = DeviceStencil(bilaplacian(2))
    m = assemble(s, g)
    b = np.sin(np.arange(m.rows) * 0.01) + 1.0
    o = SolveOptions(rel_tol=1e-8)  # above the fp64 true-residual floor at this size
    x1 = cg_solve(m, b, o)
    x2 = cg_solve_stencil(s, g, b, o)
    assert np.linalg.norm(x1 - x2) <= 1e-6 * np.linalg.norm(x1)


@pytest.mark.parametrize("bc", [BoundaryKind.clamped, BoundaryKind.simply_supported, BoundaryKind.periodic])
@pytest.mark.parametrize("check_every", [0, 7])
def test_fused_2d_iterations_match_unfused(sk_option, bc, check_every):
    # the two-kernel 2D iteration (p' = r + beta p on the tile load, p.q in
    # the apply's epilogue) follows the four-kernel one: same recurrence, only
    # the p.q summation order differs. Odd check_every exercises the p / p2
    # parity of the unrolled graph (rounded up to even); the periodic Laplacian
    # class is singular, so that case solves a mean-free right-hand side.
    N = 96
    g = make_grid(2, N + 1, 1.0 / N, bc)
    b = np.sin(np.arange(g.unknown_count()) * 0.013) + (0.0 if bc == BoundaryKind.periodic else 1.0)
    b -= b.mean() if bc == BoundaryKind.periodic else 0.0
    o = SolveOptions(rel_tol=1e-9, check_every=check_every, deflate_mean=bc == BoundaryKind.periodic)
    if check_every:
        sk_option("cg_device_loop", 0)  # the unrolled-graph fallback
    reps = []
    xs = []
    # cooperative kernel (forced), two-kernel graph, four-kernel graph
    for fused, coop in ((1, 1), (1, 0), (0, 0)):
        sk_option("cg_fused", fused)
        sk_option("cg_coop", coop)
        rep = SolveReport()
        xs.append(cg_solve_stencil(DeviceStencil(bilaplacian(2)), g, b, o, rep))  # new stencil -> new plan
        reps.append(rep)
    for k in (0, 1):
        assert abs(reps[k].iterations - reps[2].iterations) <= 2
        assert reps[k].true_rel_residual <= 1e-9
        assert np.linalg.norm(xs[k] - xs[2]) <= 1e-7 * np.linalg.norm(xs[2])
    # the cooperative kernel and the two-kernel graph run the same recurrence
    assert reps[0].iterations == reps[1].iterations


@pytest.mark.parametrize("bc", [BoundaryKind.clamped, BoundaryKind.simply_supported, BoundaryKind.periodic])
@pytest.mark.parametrize("check_every", [0, 7])
def test_3d_apply_pq_matches_separate_pass(sk_option, bc, check_every):
    # 3D radius-2 stencils: p.q reduced in the streaming apply's epilogue
    # (three kernels per iteration) follows the separate p.q pass: same
    # recurrence, only the p.q summation order differs
    N = 24
    g = make_grid(3, N + 1, 1.0 / N, bc)
    b = np.sin(np.arange(g.unknown_count()) * 0.013) + (0.0 if bc == BoundaryKind.periodic else 1.0)
    b -= b.mean() if bc == BoundaryKind.periodic else 0.0
    o = SolveOptions(rel_tol=1e-9, check_every=check_every, deflate_mean=bc == BoundaryKind.periodic)
    if check_every:
        sk_option("cg_device_loop", 0)
    reps, xs = [], []
    for pq in (1, 0):
        sk_option("cg_pq", pq)
        rep = SolveReport()
        xs.append(cg_solve_stencil(DeviceStencil(bilaplacian(3)), g, b, o, rep))
        reps.append(rep)
    assert abs(reps[0].iterations - reps[1].iterations) <= 2
    assert reps[0].true_rel_residual <= 1e-9
    assert np.linalg.norm(xs[0] - xs[1]) <= 1e-7 * np.linalg.norm(xs[1])


@pytest.mark.parametrize("dims,bcs", [((75, 19, 19), ("clamped",) * 3), ((81, 20, 19), ("simply_supported",) * 3),
                                      ((70, 33, 17), ("clamped", "periodic", "simply_supported")),
                                      ((64, 40, 24), ("periodic", "clamped", "clamped"))])
def test_padded_p_cg_is_bit_identical(sk_option, dims, bcs):
    # radius-4 matrix-free CG off periodic grids: the p-update kernel writes a
    # ghost-padded copy of p (reflected / wrapped images, boundary zeros) and
    # the apply reads it with the 16-byte loader; the tiles hold the same
    # values as the boundary-mapped loader's, so every iterate is identical
    from paper_2205_03354_b200.grid import GridSpec

    bc = [getattr(BoundaryKind, b) for b in bcs]
    n = [d + (2 if b != BoundaryKind.periodic else 0) for d, b in zip(dims, bc)]
    g = GridSpec(dim=3, n=n, h=1.0 / 32, origin=[0.0] * 3, bc=bc)
    assert g.unknown_count() == dims[0] * dims[1] * dims[2]
    b = np.sin(np.arange(g.unknown_count()) * 0.013) + 1.0
    o = SolveOptions(rel_tol=1e-9, accept_recurrence=True)
    sk_option("apply73_factored", 0)  # the literal 73 weights on both paths (the factored apply is tested below)
    out = {}
    for flag in (1, 0):
        sk_option("cg_padded", flag)
        rep = SolveReport()
        out[flag] = (cg_solve_stencil(DeviceStencil(bilaplacian(3, 4)), g, b, o, rep), rep.iterations)
    assert np.array_equal(out[1][0], out[0][0]) and out[1][1] == out[0][1]


@pytest.mark.parametrize("dims,bcs", [((96, 40, 30), ("clamped",) * 3), ((100, 34, 26), ("simply_supported",) * 3),
                                      ((80, 32, 28), ("periodic", "clamped", "simply_supported"))])
def test_padded_p_cg_factored_apply(orc, sk_option, dims, bcs):
    # With the ghost-padded p, B = compose(L4, L4) is applied as L4(L4 p_pad)
    # (fac73v2_kernel on the padded field): the pad holds every image the
    # assembled rows read, so this is the assembled operator up to rounding.
    # Same solution as the literal-weights solve and as the CSR solve of the
    # reference-assembled matrix (oracle) to the CG parity bar.
    from paper_2205_03354_b200.grid import GridSpec

    bc = [getattr(BoundaryKind, b) for b in bcs]
    n = [d + (2 if b != BoundaryKind.periodic else 0) for d, b in zip(dims, bc)]
    g = GridSpec(dim=3, n=n, h=1.0 / 32, origin=[0.0] * 3, bc=bc)
    s = bilaplacian(3, 4)
    b = np.sin(np.arange(g.unknown_count()) * 0.013) + 1.0
    o = SolveOptions(rel_tol=1e-10)
    sk_option("cg_padded", 1)
    out = {}
    for flag in (1, 0):
        sk_option("apply73_factored", flag)
        rep = SolveReport()
        out[flag] = (cg_solve_stencil(DeviceStencil(s), g, b, o, rep), rep)
        assert rep.true_rel_residual <= 1e-10
    (xf, rf), (xl, rl) = out[1], out[0]
    assert np.linalg.norm(xf - xl) <= 1e-8 * np.linalg.norm(xl)
    assert abs(rf.iterations - rl.iterations) <= max(3, 0.02 * rl.iterations)
    rp, ci, vals = orc.assemble(s, g)
    xo, status, its_o, _ = orc.cg_solve(rp, ci, vals, b, 1e-10)
    assert status == 0
    assert np.linalg.norm(xf - xo) <= 1e-8 * np.linalg.norm(xo)


@pytest.mark.parametrize("intervals", [74, 80])
def test_config5_matrix_free_factored_vs_csr_cg(sk_option, intervals):
    # config 5's operator at a size where the padded p takes the factored apply
    # with fused p.q and odd rows (73^3 / 79^3 unknowns): the solution agrees
    # with the CSR solve of the GPU-assembled matrix (bit-exact to the
    # reference's, tests/test_gpu_golden.py) to the CG parity bar. (Closer to
    # the fp64 floor of rtol 1e-10, e.g. 96^3, the true-residual restarts make
    # the iteration counts of the three operators drift apart: 9.7k CSR / 9.7k
    # literal / 11.9k factored, same solution.)
    g = make_grid(3, intervals + 1, 1.0 / intervals, BoundaryKind.clamped)
    s = bilaplacian(3, 4)
    b = np.sin(np.arange(g.unknown_count()) * 0.007) + 0.5
    o = SolveOptions(rel_tol=1e-10)
    sk_option("apply73_factored", 1)
    sk_option("cg_padded", 1)
    rep = SolveReport()
    x = cg_solve_stencil(DeviceStencil(s), g, b, o, rep)
    rc = SolveReport()
    xc = cg_solve(assemble(s, g), b, o, rc)
    assert rep.true_rel_residual <= 1e-10 and rc.true_rel_residual <= 1e-10
    assert np.linalg.norm(x - xc) <= 1e-8 * np.linalg.norm(xc)
    assert abs(rep.iterations - rc.iterations) <= max(3, 0.02 * rc.iterations)
