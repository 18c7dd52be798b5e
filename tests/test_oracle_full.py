"""Pins of the oracle's full-matrix CFD variant with a Cerjan layer (SURVEY §8f row
f4; readings F1-F2 in oracle/adi_oracle.c and DESIGN.md §3).

* dt = 0 turns the step into the pure taper: every field times G(x) G(y), with
  G(k) = exp(-(a (nb - d_k))^2) inside the layer (Cerjan et al.'s profile).
* The stage's fixed point equals the dense solve of [[I, αD], [βD, I]] with the
  full D = P^-1 Q on all n+1 nodes (a different algorithm).
* The step is linear, maps zero to zero and commutes with x / y reflection.
* Absorption: a centred pulse leaves the grid (energy < 1 % after it crosses the
  layer), while the reduced (Dirichlet) variant keeps > 50 % of it.
"""
import numpy as np
import pytest

import oracle
from adi_inputs import CFD


def _pulse(n, w=0.04):
    x = np.linspace(0, 1, n)
    X, Y = np.meshgrid(x, x)
    return np.exp(-((X - 0.5) ** 2 + (Y - 0.5) ** 2) / (2 * w * w))


def _rand(n, seed):
    r = np.random.default_rng(seed)
    return r.standard_normal((n, n)), r.standard_normal((n, n)), r.standard_normal((n, n))


def test_zero_dt_is_the_cerjan_taper():
    n, nb, a = 40, 9, 0.05
    U, V, W = _rand(n, 1)
    Uo, Vo, Wo = oracle.run_full(n, n, 1 / (n - 1), 0.0, 1.0, 8, U, V, W, nsteps=1, nb=nb, a=a)
    d = np.minimum(np.arange(n), n - 1 - np.arange(n))
    g = np.where(d < nb, np.exp(-(a * (nb - d)) ** 2), 1.0)
    G = np.outer(g, g)
    np.testing.assert_allclose(Uo, G * U, rtol=1e-15, atol=0)
    np.testing.assert_allclose(Vo, G * V, rtol=1e-15, atol=0)
    np.testing.assert_allclose(Wo, G * W, rtol=1e-15, atol=0)


@pytest.mark.parametrize("n", [8, 12, 17])
def test_full_stage_converges_to_dense_solve(n):
    """Fixed point of the oracle's full stage (K = 200) == the dense solve of
    [[I, αD], [βD, I]] [u; v] = [s; v0], D = P^-1 Q assembled column by column."""
    h = 1.0 / n
    D = np.stack([oracle.apply_D(CFD, n, h, np.eye(n + 1)[j]) for j in range(n + 1)], axis=1)
    al, be = 0.25 * h, 0.2 * h
    rng = np.random.default_rng(n)
    s, v0 = rng.standard_normal(n + 1), rng.standard_normal(n + 1)
    A = np.block([[np.eye(n + 1), al * D], [be * D, np.eye(n + 1)]])
    x = np.linalg.solve(A, np.concatenate([s, v0]))
    u, v = oracle.stage_line_full(n, h, 200, al, be, s, v0)
    np.testing.assert_allclose(np.concatenate([u, v]), x, rtol=0, atol=1e-12 * np.abs(x).max())


def test_linear_zero_and_reflection():
    n = 21
    h, dt = 1 / (n - 1), 0.5 / (n - 1)
    A = _rand(n, 2)
    B = _rand(n, 3)
    run = lambda F, **k: oracle.run_full(n, n, h, dt, 1.0, 8, *F, nsteps=3, nb=5, a=0.1, **k)
    z = run([np.zeros((n, n))] * 3)
    assert not any(x.any() for x in z)
    ra, rb = run(A), run(B)
    comb = run([0.7 * x - 1.3 * y for x, y in zip(A, B)])
    for c, x, y in zip(comb, ra, rb):
        np.testing.assert_allclose(c, 0.7 * x - 1.3 * y, rtol=0, atol=1e-12 * np.abs(c).max())
    # x-reflection: U, W even, V odd (D is centro-antisymmetric)
    Ar = (A[0][:, ::-1], -A[1][:, ::-1], A[2][:, ::-1])
    rr = run(Ar)
    np.testing.assert_allclose(rr[0], ra[0][:, ::-1], rtol=0, atol=1e-12 * np.abs(ra[0]).max())
    np.testing.assert_allclose(rr[1], -ra[1][:, ::-1], rtol=0, atol=1e-12 * np.abs(ra[1]).max())
    np.testing.assert_allclose(rr[2], ra[2][:, ::-1], rtol=0, atol=1e-12 * np.abs(ra[2]).max())


def test_cerjan_layer_absorbs():
    n, steps = 129, 220
    h = 1 / (n - 1)
    dt = 0.5 * h
    U0 = _pulse(n)
    Z = np.zeros((n, n))
    e0 = np.sum(U0 ** 2)
    U, V, W = oracle.run_full(n, n, h, dt, 1.0, 8, U0, Z, Z, nsteps=steps, nb=20, a=0.015)
    e_full = np.sum(U ** 2 + V ** 2 + W ** 2)
    # the reduced (Dirichlet) CFD variant on the same pulse: reflecting walls
    Ur, Vr, Wr = oracle.run(CFD, n, n, h, dt, 1.0, 8, U0, Z[1:-1, :], Z[:, 1:-1], nsteps=steps)
    e_red = np.sum(Ur ** 2) + np.sum(Vr ** 2) + np.sum(Wr ** 2)
    assert e_full < 0.01 * e0, e_full / e0
    assert e_red > 0.5 * e0, e_red / e0


@pytest.mark.parametrize("nsteps", [1, 4])
def test_full_variant_is_consistent(nsteps):
    """No boundary data: the full operators carry the boundary.  On a manufactured
    solution that is nonzero on the boundary (Γ = 1, k = 2, λ = 1/2), the max error of
    U, V, W after a few steps falls at order >= 2.8 from N = 32 to 256 (over long
    horizons the literal CFD closure's growth, G20, dominates: DESIGN.md §8.4)."""
    import math
    from adi_inputs import MMS
    case = MMS(gamma=1.0, k=2, lam=0.5)
    errs = []
    for N in (32, 64, 128, 256):
        n, h = N + 1, 1.0 / N
        dt = 0.5 * h
        x = np.linspace(0, 1, n)
        X, Y = np.meshgrid(x, x)
        Z = np.zeros((n, n))
        gf = np.sin(case.omega * np.arange(2 * nsteps + 1) * dt / 2)
        U, V, W = oracle.run_full(n, n, h, dt, 1.0, 8, case.S(X, Y), Z, Z, phi=case.phi(X, Y), gf=gf,
                                  nsteps=nsteps)
        t = nsteps * dt
        errs.append(max(np.abs(U - case.u(X, Y, t)).max(), np.abs(V - case.v(X, Y, t)).max(),
                        np.abs(W - case.w(X, Y, t)).max()))
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(3)]
    assert all(r >= 2.8 for r in rates), (errs, rates)
