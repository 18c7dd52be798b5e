"""Pins for the oracle's ADI stage and step (eqs. 5-9, Alg. 1-4).

* Stage: K -> large converges to the direct (dense LU) solution of the coupled
  line system of eq. 7 — a different algorithm.
* Step: exact zero fixed point, linearity in (state, source, boundary),
  reflection commutation (centro-antisymmetric operators), MFD stability at
  the paper's cfl_max = 0.81 and blow-up above the inner-iteration limit.
"""
import numpy as np
import pytest

import oracle
from adi_inputs import CFD, MFD, random_problem


def _run(p, nsteps, **over):
    kw = p.oracle_kwargs()
    kw.update(over)
    return oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=nsteps, **kw)


def _dense(method, n, h):
    nv = n + 1
    nub = n + 1 if method == CFD else n + 2
    Db = np.stack([oracle.apply_Dbar(method, n, h, np.eye(nv)[j]) for j in range(nv)], axis=1)
    D = np.stack([oracle.apply_D(method, n, h, np.eye(nub)[j]) for j in range(nub)], axis=1)
    return Db, D


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n", [8, 12, 16])
def test_stage_converges_to_direct_solve(method, n):
    """Fixed point of eq. 8 == solution of [[I, αD̄], [βD_int, I]] [u; v] = [s; v0 - βD_bnd g]."""
    h = 1.0 / n
    dt = 0.5 * h
    alpha = beta = dt / 2
    rng = np.random.default_rng(n + 10 * method)
    Db, D = _dense(method, n, h)
    nu, nv = Db.shape
    s = rng.standard_normal(nu)
    v0 = rng.standard_normal(nv)
    gL, gR = rng.standard_normal(2)
    A = np.block([[np.eye(nu), alpha * Db], [beta * D[:, 1:-1], np.eye(nv)]])
    rhs = np.concatenate([s, v0 - beta * (D[:, 0] * gL + D[:, -1] * gR)])
    x = np.linalg.solve(A, rhs)
    u, v = oracle.stage_line(method, n, h, 200, alpha, beta, s, v0, gL, gR)
    np.testing.assert_allclose(np.concatenate([u, v]), x, rtol=0, atol=1e-13 * np.abs(x).max())


@pytest.mark.parametrize("method", [CFD, MFD])
def test_stage_one_sweep_by_hand(method):
    """K=1 is exactly u = s - αD̄(v0); v = v0 - βD([gL,u,gR]) (eq. 8, k=0)."""
    n = 12
    h = 1.0 / n
    alpha, beta = 0.3 * h, 0.2 * h
    rng = np.random.default_rng(1)
    Db, D = _dense(method, n, h)
    s = rng.standard_normal(Db.shape[0])
    v0 = rng.standard_normal(Db.shape[1])
    u_ref = s - alpha * (Db @ v0)
    v_ref = v0 - beta * (D @ np.concatenate([[0.7], u_ref, [-0.4]]))
    u, v = oracle.stage_line(method, n, h, 1, alpha, beta, s, v0, 0.7, -0.4)
    np.testing.assert_allclose(u, u_ref, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(v, v_ref, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("method", [CFD, MFD])
def test_zero_fixed_point(method):
    p = random_problem(method, 17, steps=3)
    z = lambda a: np.zeros_like(a)
    U, V, W = oracle.run(method, p.nx, p.ny, p.h, p.dt, p.c, p.K, z(p.U), z(p.V), z(p.W), nsteps=3)
    assert not U.any() and not V.any() and not W.any()


@pytest.mark.parametrize("method", [CFD, MFD])
def test_linearity(method):
    """The step is linear in (state, source pattern, boundary pattern)."""
    p = random_problem(method, 19, seed=1, steps=2)
    q = random_problem(method, 19, seed=2, steps=2)
    a, b = 0.7, -1.3
    r1 = _run(p, 2)
    r2 = oracle.run(method, q.nx, q.ny, q.h, p.dt, p.c, p.K, q.U, q.V, q.W, nsteps=2, phi=q.phi,
                    gf=p.gf, edges=q.edges, gb=p.gb)
    comb = oracle.run(method, p.nx, p.ny, p.h, p.dt, p.c, p.K, a * p.U + b * q.U, a * p.V + b * q.V,
                      a * p.W + b * q.W, nsteps=2, phi=a * p.phi + b * q.phi, gf=p.gf,
                      edges=tuple(a * x + b * y for x, y in zip(p.edges, q.edges)), gb=p.gb)
    for X, Y, Z in zip(r1, r2, comb):
        np.testing.assert_allclose(Z, a * X + b * Y, rtol=0, atol=1e-12 * np.abs(Z).max())


def _reflect(p, axis):
    """R_x: x -> 1-x (V̄ changes sign); R_y: y -> 1-y (W̄ changes sign)."""
    y0, y1, x0, x1 = p.edges
    if axis == "x":
        return dict(U=p.U[:, ::-1], V=-p.V[:, ::-1], W=p.W[:, ::-1], phi=p.phi[:, ::-1],
                    edges=(y0[::-1], y1[::-1], x1, x0))
    return dict(U=p.U[::-1, :], V=p.V[::-1, :], W=-p.W[::-1, :], phi=p.phi[::-1, :],
                edges=(y1, y0, x0[::-1], x1[::-1]))


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("axis", ["x", "y"])
def test_reflection_commutes_with_step(method, axis):
    """step(R s) = R step(s): the operators are centro-antisymmetric (App. A/B)."""
    p = random_problem(method, 17, seed=5, steps=1)
    U, V, W = _run(p, 1)
    r = _reflect(p, axis)
    U2, V2, W2 = oracle.run(method, p.nx, p.ny, p.h, p.dt, p.c, p.K, r["U"], r["V"], r["W"],
                            nsteps=1, phi=r["phi"], gf=p.gf, edges=r["edges"], gb=p.gb)
    from types import SimpleNamespace
    out = _reflect(SimpleNamespace(U=U, V=V, W=W, phi=p.phi, edges=p.edges), axis)
    for A, B in ((U2, out["U"]), (V2, out["V"]), (W2, out["W"])):
        np.testing.assert_allclose(A, B, rtol=0, atol=1e-13 * np.abs(B).max())


def _norm(U, V, W):
    return np.sqrt((U[1:-1, 1:-1] ** 2).sum() + (V ** 2).sum() + (W ** 2).sum())


def test_mfd_stable_at_cfl_max():
    """MFD at the paper's cfl_max = 0.81 stays bounded over 1000
    steps (zero source, homogeneous Dirichlet, random data). The identity-weighted
    norm is not the conserved mimetic energy, so it oscillates."""
    p = random_problem(MFD, 33, seed=0, cfl=0.81, source=False, boundary=False)
    p.U[0, :] = p.U[-1, :] = p.U[:, 0] = p.U[:, -1] = 0
    n0 = _norm(p.U, p.V, p.W)
    U, V, W = p.U, p.V, p.W
    ratios = []
    for _ in range(10):
        U, V, W = oracle.run(MFD, p.nx, p.ny, p.h, p.dt, 1.0, 8, U, V, W, nsteps=100)
        ratios.append(_norm(U, V, W) / n0)
    assert 0.6 < min(ratios) and max(ratios) < 1.05, ratios


def test_mfd_unstable_above_iteration_limit():
    """Above cfl = 2/sqrt(6) the K-sweep iteration diverges (SURVEY SA-3/4):
    cfl 1.3 goes non-finite within a few hundred steps."""
    p = random_problem(MFD, 33, seed=0, cfl=1.3, source=False, boundary=False)
    U, V, W = oracle.run(MFD, p.nx, p.ny, p.h, p.dt, 1.0, 8, p.U, p.V, p.W, nsteps=300)
    assert not np.all(np.isfinite(U))


def test_cfd_growth_regression():
    """Documented behaviour of the literal CFD reading:
    per-step growth of the dominant mode ~1.076 at cfl 0.91, K=8, N=64.
    Regression pin only — the paper reports stable CFD runs."""
    p = random_problem(CFD, 65, seed=0, cfl=0.91, source=False, boundary=False)
    U, V, W = p.U, p.V, p.W
    U[0, :] = U[-1, :] = U[:, 0] = U[:, -1] = 0
    U, V, W = oracle.run(CFD, p.nx, p.ny, p.h, p.dt, 1.0, 8, U, V, W, nsteps=200)
    n1 = _norm(U, V, W)
    U, V, W = oracle.run(CFD, p.nx, p.ny, p.h, p.dt, 1.0, 8, U, V, W, nsteps=100)
    g = (_norm(U, V, W) / n1) ** (1 / 100)
    assert 1.06 < g < 1.09, g
