"""Pins of the oracle's inner stopping rule (Alg. 3/4,
PAPER.md:652-721: "test <- ||U_{k+1}-U_k|| + ||V_{k+1}-V_k||, until test <= eps or
k >= k_max"; sweeps before k_min untested)."""
import numpy as np
import pytest

import oracle
from adi_inputs import CFD, MFD, random_problem


def run(p, steps, **kw):
    info = {}
    out = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=steps,
                     info=info, **p.oracle_kwargs(), **kw)
    return out, info


@pytest.mark.parametrize("method", [CFD, MFD])
def test_eps_zero_is_fixed_K(method):
    p = random_problem(method, 21, seed=3, steps=2)
    a, _ = run(p, 2)
    b, info = run(p, 2, eps=0.0)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert (info["k"] == p.K).all()


@pytest.mark.parametrize("method", [CFD, MFD])
def test_huge_eps_stops_at_kmin_and_tiny_eps_at_kmax(method):
    p = random_problem(method, 21, seed=4, steps=2)
    p.K = 9
    lo, info = run(p, 2, eps=1e300, kmin=4)
    assert (info["k"] == 4).all()
    q = random_problem(method, 21, seed=4, steps=2)
    q.K = 4
    ref, _ = run(q, 2)
    for x, y in zip(lo, ref):
        assert np.array_equal(x, y)
    hi, info = run(p, 2, eps=1e-300, kmin=4)
    assert (info["k"] == 9).all()
    ref9, _ = run(p, 2)
    for x, y in zip(hi, ref9):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("method", [CFD, MFD])
def test_first_row_stage_tests_from_single_line_stages(method):
    """The first row stage's test values, recomputed from fixed-K single-line stages
    (or_stage_line, a separate code path) for K = k and k-1 over every line."""
    n = 19
    p = random_problem(method, n, seed=5, steps=1)
    p.K = 10
    kmin = 3
    N = n - 1
    kappa = p.rho * p.c ** 2
    alpha, beta = kappa * p.dt / 2, p.dt / (2 * p.rho)
    # S1 rows (a2, Alg. 1/2 line 8): U interior - alpha D̄_y(W̄) + dt/2 F(t^0)
    U, V, W = p.U, p.V, p.W
    kw = p.oracle_kwargs()
    gf0 = kw["gf"][0] if kw.get("gf") is not None else 1.0
    gbh = kw["gb"][1] if kw.get("gb") is not None else 1.0
    nyi = U.shape[0] - 2
    nxi = U.shape[1] - 2
    S1 = np.empty((nyi, nxi))
    for ii in range(nxi):
        d = oracle.apply_Dbar(method, N, p.h, W[:, ii])
        S1[:, ii] = U[1:-1, ii + 1] - alpha * d + (p.dt / 2) * kw["phi"][:, ii] * gf0
    ex0, ex1 = kw["edges"][2], kw["edges"][3]

    def stage(K):
        us, vs = [], []
        for jj in range(nyi):
            u, v = oracle.stage_line(method, N, p.h, K, alpha, beta, S1[jj], V[jj],
                                     ex0[jj + 1] * gbh, ex1[jj + 1] * gbh)
            us.append(u)
            vs.append(v)
        return np.array(us), np.array(vs)

    it = {k: stage(k) for k in range(kmin - 1, p.K + 1)}
    tests = {k: np.linalg.norm(it[k][0] - it[k - 1][0]) + np.linalg.norm(it[k][1] - it[k - 1][1])
             for k in range(kmin, p.K + 1)}
    _, info = run(p, 1, eps=1e300, kmin=kmin)
    for k in range(kmin, p.K + 1):
        assert info["tests"][0, 0, k] == pytest.approx(tests[k], rel=1e-12, abs=1e-300)
    # an eps between two consecutive test values selects the first k below it
    ks = sorted(tests)
    for k in ks[1:]:
        if tests[k] < tests[k - 1]:
            eps = np.sqrt(tests[k] * tests[k - 1])
            want = min(j for j in ks if tests[j] <= eps)
            _, info = run(p, 1, eps=eps, kmin=kmin)
            assert info["k"][0, 0] == want
            break
