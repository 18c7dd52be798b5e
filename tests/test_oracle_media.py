"""Pins of the oracle's heterogeneous-media path (K = kappa(x,y),
R = rho^-1(x,y) grid values; "K.*( )" / "R.*( )" after the
derivative in Alg. 1-4, PAPER.md:155-167, 655-696 [G8]).

* Constant fields reduce to the scalar path (bit-exact for exactly representable
  scalings, to rounding otherwise).
* Impedance scaling: (s kappa, R/s) with (U, V/s, W/s) gives the same U and
  velocities scaled by 1/s, bit for bit for s = 2 (the pressure equation carries
  kappa, the velocity equations carry R: a swap fails).
* The stage's fixed point equals the dense solve of the per-point coupled line
  system (a different algorithm).
* A manufactured solution in a smooth medium (adi_inputs.media) converges at the
  homogeneous Γ≠0 rate (≈1 in the unnormalised Frobenius norm, 2 in h-weighted
  L2); sampling R half a cell off, or swapping kappa and R, breaks it.
"""
import math

import numpy as np
import pytest

import oracle
from adi_inputs import CFD, MFD, random_problem
from adi_inputs.media import MediumMMS, medium_error, medium_mms_problem


def _run(p, steps, **over):
    kw = p.oracle_kwargs()
    kw.update(over)
    return oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=steps, **kw)


def _const_media(p, k, r):
    return dict(kappa=np.full(p.U.shape, k), rinv_v=np.full(p.V.shape, r), rinv_w=np.full(p.W.shape, r))


@pytest.mark.parametrize("method", [CFD, MFD])
def test_constant_fields_equal_scalar_path(method):
    p = random_problem(method, 19, seed=11, steps=3)
    # rho = 0.5, c = 2: kappa = rho c^2 = 2, R = 2 (exact scalings: bit-exact)
    ref = oracle.run(method, p.nx, p.ny, p.h, p.dt, 2.0, p.K, p.U, p.V, p.W, nsteps=3,
                     **{**p.oracle_kwargs(), "rho": 0.5})
    got = _run(p, 3, **_const_media(p, 2.0, 2.0))
    for a, b in zip(ref, got):
        assert np.array_equal(a, b)
    # general constants: to rounding
    c = math.sqrt(1.3 / 0.7 ** -1)
    ref = oracle.run(method, p.nx, p.ny, p.h, p.dt, c, p.K, p.U, p.V, p.W, nsteps=3,
                     **{**p.oracle_kwargs(), "rho": 1 / 0.7})
    got = _run(p, 3, **_const_media(p, 1.3, 0.7))
    for a, b in zip(ref, got):
        np.testing.assert_allclose(b, a, rtol=0, atol=1e-13 * np.abs(a).max())


@pytest.mark.parametrize("method", [CFD, MFD])
def test_impedance_scaling_is_exact(method):
    p = random_problem(method, 21, seed=12, steps=3, media=True)
    U, V, W = _run(p, 3)
    s = 2.0
    U2, V2, W2 = oracle.run(method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V / s, p.W / s, nsteps=3,
                            **{**p.oracle_kwargs(), "kappa": s * p.kappa.astype(np.float64),
                               "rinv_v": p.rinv_v / s, "rinv_w": p.rinv_w / s})
    assert np.array_equal(U2, U)
    assert np.array_equal(V2, V / s)
    assert np.array_equal(W2, W / s)
    # the swap (kappa on the velocity equations) is not invariant
    Us, _, _ = oracle.run(method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V / s, p.W / s, nsteps=3,
                          **{**p.oracle_kwargs(), "kappa": p.kappa / s,
                             "rinv_v": s * p.rinv_v.astype(np.float64), "rinv_w": s * p.rinv_w.astype(np.float64)})
    assert not np.allclose(Us, U)


@pytest.mark.parametrize("method", [CFD, MFD])
def test_boundary_entries_of_kappa_unused(method):
    p = random_problem(method, 17, seed=13, steps=2, media=True)
    a = _run(p, 2)
    k = p.kappa.astype(np.float64).copy()
    k[0, :] = k[-1, :] = k[:, 0] = k[:, -1] = 123.0
    b = _run(p, 2, kappa=k)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def _dense(method, n, h):
    nv = n + 1
    nub = n + 1 if method == CFD else n + 2
    Db = np.stack([oracle.apply_Dbar(method, n, h, np.eye(nv)[j]) for j in range(nv)], axis=1)
    D = np.stack([oracle.apply_D(method, n, h, np.eye(nub)[j]) for j in range(nub)], axis=1)
    return Db, D


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n", [8, 13])
def test_stage_with_fields_converges_to_direct_solve(method, n):
    """Fixed point of u = s - a∘D̄v, v = v0 - b∘D[gL,u,gR] == dense solve of
    [[I, diag(a) D̄], [diag(b) D_int, I]] [u; v] = [s; v0 - diag(b) D_bnd g]."""
    h = 1.0 / n
    dt = 0.5 * h
    rng = np.random.default_rng(7 * n + method)
    Db, D = _dense(method, n, h)
    nu, nv = Db.shape
    a = dt / 2 * rng.uniform(0.5, 1.0, nu)
    b = dt / 2 * rng.uniform(0.5, 1.0, nv)
    s = rng.standard_normal(nu)
    v0 = rng.standard_normal(nv)
    gL, gR = rng.standard_normal(2)
    A = np.block([[np.eye(nu), a[:, None] * Db], [b[:, None] * D[:, 1:-1], np.eye(nv)]])
    rhs = np.concatenate([s, v0 - b * (D[:, 0] * gL + D[:, -1] * gR)])
    x = np.linalg.solve(A, rhs)
    u, v = oracle.stage_line(method, n, h, 200, a, b, s, v0, gL, gR)
    np.testing.assert_allclose(np.concatenate([u, v]), x, rtol=0, atol=1e-13 * np.abs(x).max())


def _mms_errors(mutate=None, Ns=(32, 64, 128)):
    errs = []
    for N in Ns:
        p = medium_mms_problem(MFD, N + 1, t_sim=MediumMMS().T)
        kw = p.oracle_kwargs()
        if mutate:
            mutate(p, kw)
        U, _, _ = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W,
                             nsteps=p.meta["steps"], **kw)
        errs.append(medium_error(p, U, p.meta["t_end"]))
    return errs, [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]


def test_medium_mms_converges():
    errs, rates = _mms_errors()
    assert errs[-1] < 0.2
    assert all(r >= 0.9 for r in rates), rates


def test_medium_mms_detects_misplaced_R():
    """R sampled half a cell off the V̄ points loses the rate (the pin discriminates)."""
    from adi_inputs.grid import Grid
    m = MediumMMS().medium

    def shift(p, kw):
        xv, yv = Grid(MFD, p.nx, p.ny).v_xy()
        kw["rinv_v"] = m.R(xv[None, :] + 0.5 * p.h, yv[:, None])

    _, rates = _mms_errors(shift)
    assert rates[-1] < 0.8, rates
