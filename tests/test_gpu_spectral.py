"""Spectral tools on the device: power_iteration and
periodic_spectrum (linalg.cpp:74-106, 149-222), against the reference's own
known answers (test_linalg.cpp:74-145, exact dyadic rows included) and the
oracle restatement."""
import numpy as np
import pytest

from paper_2205_03354_b200.errors import StencilkitError
from paper_2205_03354_b200.grid import BoundaryKind, DeviceStencil, GridSpec, assemble, make_grid, make_periodic_grid
from paper_2205_03354_b200.linalg import periodic_spectrum, power_iteration
from paper_2205_03354_b200.stencil import Stencil, StencilSpec, bilaplacian, builtin_stencil, laplacian, make

pytestmark = pytest.mark.gpu


def test_power_iteration_known_answers():
    # test_linalg.cpp:74-84
    g = make_periodic_grid(2, 8, 1.0)
    eye = assemble(DeviceStencil(Stencil.identity(2)), g)
    assert power_iteration(eye, 1e-10) == pytest.approx(1.0, rel=1e-9)
    g20 = make_periodic_grid(2, 20, 10.0)
    bil = builtin_stencil("bilaplacian-2d")
    rho = power_iteration(assemble(DeviceStencil(bil), g20), 1e-8)
    assert rho == pytest.approx(periodic_spectrum(bil, g20).spectral_radius, rel=1e-6)


def test_spectrum_1d_laplacian_modes():
    # test_linalg.cpp:86-95
    g = make_periodic_grid(1, 4, 0.5)
    rep = periodic_spectrum(make(StencilSpec(2, 2)), g)
    assert rep.eigenvalues.size == 4
    assert rep.eigenvalues[0].real == pytest.approx(0.0, abs=1e-14)
    assert rep.eigenvalues[1].real == pytest.approx(-8.0, rel=1e-13)
    assert rep.eigenvalues[2].real == pytest.approx(-16.0, rel=1e-13)
    assert rep.spectral_radius == pytest.approx(16.0, rel=1e-13)


def test_spectrum_requires_periodic():
    g = make_grid(1, 8, 1.0, BoundaryKind.simply_supported)
    with pytest.raises(StencilkitError):
        periodic_spectrum(Stencil.identity(1), g)


@pytest.mark.parametrize("h,dt,rho,rho_step", [(8, 2, 0.015625, 1.03125), (4, 1, 0.25, 1.25), (2, 0.5, 4.0, 3.0),
                                               (1, 0.25, 64.0, 17.0)])
def test_time_stepping_table_rows(h, dt, rho, rho_step):
    # test_linalg.cpp:107-145: exact dyadic radii on [0, 200]^2
    bil = builtin_stencil("bilaplacian-2d")
    n = int(200.0 / h)
    g = make_periodic_grid(2, n, float(h))
    b = periodic_spectrum(bil, g)
    assert b.symbol_radius == rho
    if n % 2 == 0:
        assert b.spectral_radius == rho
    step = periodic_spectrum(bil, g, 1.0, dt)
    assert step.symbol_radius == rho_step
    if n % 2 == 0:
        assert step.spectral_radius == rho_step
        assert step.condition_estimate == rho_step
    # the reference's test asserts imag == 0.0 exactly; the compiled reference
    # itself (no FMA contraction) leaves ~1e-19 here, as does the device
    assert np.all(np.abs(b.eigenvalues.imag) <= 1e-15 * rho)
    assert np.all(b.eigenvalues.real >= -1e-13)


def test_odd_grid_radius():
    bil = builtin_stencil("bilaplacian-2d")
    b25 = periodic_spectrum(bil, make_periodic_grid(2, 25, 8.0))
    assert b25.spectral_radius == pytest.approx(0.0155018, rel=1e-4)
    assert b25.spectral_radius < b25.symbol_radius


@pytest.mark.parametrize("dim,acc,n,h", [(2, 2, (40, 24), 0.5), (3, 2, (12, 10, 9), 1.0), (2, 4, (30, 30), 1.0),
                                         (3, 4, (16, 16, 16), 0.25)])
def test_spectrum_vs_oracle(orc, dim, acc, n, h):
    s = bilaplacian(dim, acc)
    g = GridSpec(dim=dim, n=list(n), h=h, origin=[0.0] * dim, bc=[BoundaryKind.periodic] * dim)
    for shift, scale in [(0.0, 1.0), (1.0, 1e-3)]:
        rep = periodic_spectrum(s, g, shift, scale)
        e, rho, cond = orc.periodic_eigen(s, g, shift, scale)
        assert np.max(np.abs(rep.eigenvalues - e)) <= 1e-13 * rho
        assert rep.spectral_radius == pytest.approx(rho, rel=1e-14)
        assert rep.condition_estimate == pytest.approx(cond, rel=1e-12)
        assert rep.symbol_radius >= rep.spectral_radius * (1 - 1e-14)


def test_power_iteration_vs_oracle(orc):
    for dim, n, h in [(2, 24, 1.0), (3, 9, 0.5)]:
        g = make_periodic_grid(dim, n, h)
        s = laplacian(dim, 2)
        m = assemble(DeviceStencil(s), g)
        lam = power_iteration(m, 1e-9)
        ref, _ = orc.power_iteration(*orc.assemble(s, g), 1e-9)
        assert lam == pytest.approx(ref, rel=1e-8)
        assert lam == pytest.approx(periodic_spectrum(s, g).spectral_radius, rel=1e-7)
