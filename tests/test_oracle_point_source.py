"""Pins for the oracle's point source (``source_at`` / ``source_full`` in
oracle/adi_oracle.c), independent of the oracle's own arithmetic.

The source term f of eq. 1 enters the scheme as the A_F term of
eqs. 5-6: Δt/2 F(t^m) in stage 1 and Δt/2 F(t^{m+1}) in stage 2.
A point source is the discrete delta F = g_f(t)/h^2 at one pressure point
(SURVEY §8a-a7, §8d item 5).  Three facts fix it without re-typing its formula:

* **Mass.** With zero initial data, ``∫ u dx`` grows by ``∫ f dx dt`` as long as
  the velocities vanish near the boundary (the derivative operators of App. A/B
  telescope on compactly supported data: their interior rows sum to zero).  For
  F = g/h^2 at one point, h^2 Σ U after m steps must equal the trapezoid
  Σ_k Δt/2 (g(t_k) + g(t_{k+1})) of the time function — a closed form.  A missing
  or doubled 1/h^2, or a source entering only one stage, fails it.
* **Position.** A source at the centre of the grid, from zero data, gives a field
  symmetric under x- and y-reflection (the step commutes with reflection,
  ``test_oracle_step.test_reflection_commutes_with_step``).  An index off by one
  (U index vs interior index) moves the source off the centre and breaks the
  symmetry (the mutation check below shows the test would see it).
* **Equivalence.** At any (ix, iy), the point source equals the dense-source path
  with φ = e_{(iy-1, ix-1)} / h^2 (the dense path is pinned by the MMS rates,
  ``test_oracle_mms``), with random state, boundary data and time tables.
"""
import numpy as np
import pytest

import oracle
from adi_inputs import CFD, MFD, shapes, interior_shape


def _zero_run(method, n, src, gf, steps, K=8, cfl=None):
    h = 1.0 / (n - 1)
    cfl = cfl if cfl is not None else (0.91 if method == CFD else 0.81)
    dt = cfl * h
    su, sv, sw = shapes(method, n, n)
    out = oracle.run(method, n, n, h, dt, 1.0, K, np.zeros(su), np.zeros(sv), np.zeros(sw),
                     src=src, gf=gf, nsteps=steps)
    return h, dt, out


def _centre(method, n):
    """U index of the grid centre: CFD node (n-1)/2 (n odd); MFD cell-centre
    (X_cb) index (N+1)/2 with N = n-1 cells (n even), i.e. x = 1/2 in both."""
    if method == CFD:
        assert n % 2 == 1
        return (n - 1) // 2
    assert n % 2 == 0
    return n // 2


def _trapezoid(gf, dt, steps):
    return sum(dt / 2.0 * (gf[2 * k] + gf[2 * k + 2]) for k in range(steps))


@pytest.mark.parametrize("method,n", [(CFD, 129), (MFD, 128)])
def test_point_source_mass(method, n):
    """h^2 Σ U = ∫ g dt (trapezoid at the step times) while the field is far from
    the boundary: two steps of a centred source on a grid with 63 cells of margin."""
    rng = np.random.default_rng(3)
    steps = 2
    gf = rng.uniform(0.5, 1.5, 2 * steps + 1)
    c = _centre(method, n)
    h, dt, (U, V, W) = _zero_run(method, n, (c, c), gf, steps)
    mass = h * h * U[1:-1, 1:-1].sum()
    expect = _trapezoid(gf, dt, steps)
    assert abs(mass - expect) <= 1e-12 * abs(expect), (mass, expect)
    # the scaling is what is pinned: without the 1/h^2 the mass would be h^2 smaller
    assert abs(mass * h * h - expect) > 0.5 * abs(expect)
    # the field really spread (the test is not trivially the source itself)
    assert np.count_nonzero(np.abs(U) > 1e-6 * np.abs(U).max()) > 100


def test_point_source_mass_full_variant():
    """The same closed form for the full-matrix variant (NEXT row f4, run_full): every
    node is unknown and the source may sit on any node; no Cerjan layer."""
    n = 129
    rng = np.random.default_rng(4)
    steps = 2
    gf = rng.uniform(0.5, 1.5, 2 * steps + 1)
    h = 1.0 / (n - 1)
    dt = 0.91 * h
    z = np.zeros((n, n))
    c = (n - 1) // 2
    U, V, W = oracle.run_full(n, n, h, dt, 1.0, 8, z, z, z, src=(c, c), gf=gf, nsteps=steps)
    mass = h * h * U.sum()
    expect = _trapezoid(gf, dt, steps)
    assert abs(mass - expect) <= 1e-12 * abs(expect), (mass, expect)


def _sym_err(U, V, W):
    """Deviation from the reflection symmetry of a centred source (R_x, R_y of
    test_oracle_step: U even, V̄ odd in x, W̄ odd in y), relative to max |U|."""
    s = np.abs(U).max()
    e = max(np.abs(U - U[:, ::-1]).max(), np.abs(U - U[::-1, :]).max(),
            np.abs(V + V[:, ::-1]).max(), np.abs(V - V[::-1, :]).max(),
            np.abs(W - W[:, ::-1]).max(), np.abs(W + W[::-1, :]).max())
    return e / s


@pytest.mark.parametrize("method,n", [(CFD, 33), (MFD, 34)])
def test_point_source_centred_is_symmetric(method, n):
    """From zero data, a source at the centre keeps the field reflection-symmetric;
    an off-by-one source (mutation) does not."""
    rng = np.random.default_rng(5)
    steps = 6
    gf = rng.standard_normal(2 * steps + 1)
    c = _centre(method, n)
    _, _, out = _zero_run(method, n, (c, c), gf, steps)
    assert _sym_err(*out) <= 1e-13
    for src in ((c + 1, c), (c, c - 1)):
        _, _, bad = _zero_run(method, n, src, gf, steps)
        assert _sym_err(*bad) > 1e-3


def test_point_source_centred_is_symmetric_full_variant():
    n = 33
    rng = np.random.default_rng(6)
    steps = 6
    gf = rng.standard_normal(2 * steps + 1)
    h = 1.0 / (n - 1)
    z = np.zeros((n, n))
    c = (n - 1) // 2
    for nb in (0, 6):
        U, V, W = oracle.run_full(n, n, h, 0.91 * h, 1.0, 8, z, z, z, src=(c, c), gf=gf, nsteps=steps, nb=nb)
        s = np.abs(U).max()
        assert max(np.abs(U - U[:, ::-1]).max(), np.abs(U - U[::-1, :]).max(),
                   np.abs(V + V[:, ::-1]).max(), np.abs(W + W[::-1, :]).max()) <= 1e-13 * s
        U2, _, _ = oracle.run_full(n, n, h, 0.91 * h, 1.0, 8, z, z, z, src=(c + 1, c), gf=gf, nsteps=steps, nb=nb)
        assert np.abs(U2 - U2[:, ::-1]).max() > 1e-3 * np.abs(U2).max()


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("where", ["inner", "corner"])
def test_point_source_equals_dense_delta(method, where):
    """src = (ix, iy) == the dense path with φ = e_{(iy-1, ix-1)} / h^2, from a random
    state with random boundary data (the same run otherwise)."""
    n = 27
    rng = np.random.default_rng(7 + method)
    steps = 3
    h = 1.0 / (n - 1)
    dt = (0.91 if method == CFD else 0.81) * h
    su, sv, sw = shapes(method, n, n)
    ni = interior_shape(method, n, n)
    U, V, W = rng.standard_normal(su), rng.standard_normal(sv), rng.standard_normal(sw)
    edges = (rng.standard_normal(su[1]), rng.standard_normal(su[1]), rng.standard_normal(su[0]),
             rng.standard_normal(su[0]))
    gf = rng.standard_normal(2 * steps + 1)
    gb = rng.standard_normal(2 * steps + 1)
    ix, iy = (9, 14) if where == "inner" else (1, ni[0])   # U indices; "corner": first column, last row
    kw = dict(edges=edges, gb=gb, gf=gf, nsteps=steps)
    pt = oracle.run(method, n, n, h, dt, 1.0, 8, U, V, W, src=(ix, iy), **kw)
    phi = np.zeros(ni)
    phi[iy - 1, ix - 1] = 1.0 / (h * h)
    dense = oracle.run(method, n, n, h, dt, 1.0, 8, U, V, W, phi=phi, **kw)
    for a, b in zip(pt, dense):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-13 * np.abs(b).max())
    # mutation: the delta one interior index off (the U-vs-interior confusion) differs
    phi2 = np.zeros(ni)
    phi2[iy - 1, ix - 1 + (1 if ix < ni[1] else -1)] = 1.0 / (h * h)
    off = oracle.run(method, n, n, h, dt, 1.0, 8, U, V, W, phi=phi2, **kw)
    assert np.abs(off[0] - pt[0]).max() > 1e-3 * np.abs(pt[0]).max()


def test_point_source_equals_dense_delta_full_variant():
    n = 27
    rng = np.random.default_rng(9)
    steps = 3
    h = 1.0 / (n - 1)
    U, V, W = (rng.standard_normal((n, n)) for _ in range(3))
    gf = rng.standard_normal(2 * steps + 1)
    for ix, iy in ((0, 0), (11, 20), (n - 1, 5)):   # any node, boundary nodes included
        pt = oracle.run_full(n, n, h, 0.91 * h, 1.0, 8, U, V, W, src=(ix, iy), gf=gf, nsteps=steps, nb=5)
        phi = np.zeros((n, n))
        phi[iy, ix] = 1.0 / (h * h)
        dense = oracle.run_full(n, n, h, 0.91 * h, 1.0, 8, U, V, W, phi=phi, gf=gf, nsteps=steps, nb=5)
        for a, b in zip(pt, dense):
            np.testing.assert_allclose(a, b, rtol=0, atol=1e-13 * np.abs(b).max())
