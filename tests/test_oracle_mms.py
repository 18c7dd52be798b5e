"""Pins against the paper's exact solution (eq. 11) and its convergence study.

* The MMS fields satisfy eq. 1 (finite-difference residual).
* MFD on the Γ=0 harmonic problem converges at a rate near 4
  (abstract; Table 4) and near 2 on the
  Γ=k=2 boundary-gradient problem.
* CFD at a short horizon converges at the O(Δt²) time-error rate (the literal
  CFD reading is unstable over 5T: DESIGN.md §3).
* The rate harness reproduces the printed trimmed averages of Tables 3-4.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
from adi_inputs import (CFD, MFD, MMS, dt_for_cfl, dt_rate_study, estimate_rates, mms_problem,
                        trimmed_average)
from adi_inputs.mms import interior_error
from conftest import read_golden

T = 1.0 / math.sqrt(2.0)


@pytest.mark.parametrize("case", [MMS(), MMS(gamma=2, k=2), MMS(gamma=9, k=9),
                                  MMS(gamma=2, k=2, kappa=2.25, rho=1.0)])
def test_mms_fields_satisfy_pde(case):
    """u_t = -κ(v_x + w_y) + f and ρ v_t = -u_x, ρ w_t = -u_y (eq. 1)
    at 100 random points, 4th-order central differences."""
    rng = np.random.default_rng(7)
    d = 1e-3
    c4 = lambda F, z: (-F(z + 2 * d) + 8 * F(z + d) - 8 * F(z - d) + F(z - 2 * d)) / (12 * d)
    worst = 0.0
    for _ in range(100):
        x, y, t = rng.uniform(0.05, 0.95), rng.uniform(0.05, 0.95), rng.uniform(0, 2)
        ut = c4(lambda s: case.u(x, y, s), t)
        div = c4(lambda s: case.v(s, y, t), x) + c4(lambda s: case.w(x, s, t), y)
        r1 = ut + case.kappa * div - case.f(x, y, t)
        r2 = case.rho * c4(lambda s: case.v(x, y, s), t) + c4(lambda s: case.u(s, y, t), x)
        r3 = case.rho * c4(lambda s: case.w(x, y, s), t) + c4(lambda s: case.u(x, s, t), y)
        scale = 1.0 + abs(case.f(x, y, t)) + abs(ut)
        worst = max(worst, abs(r1) / scale, abs(r2) / scale, abs(r3) / scale)
    assert worst < 1e-6, worst


def test_spec_examples():
    ex = {r[0]: r[1:] for r in read_golden("spec_examples.txt")}
    assert dt_for_cfl(1 / 16, 0.91) == pytest.approx(float(ex["dt_cfd_N16"][0]), abs=1e-15)
    assert dt_for_cfl(1 / 16, 0.81) == pytest.approx(float(ex["dt_mfd_N16"][0]), abs=1e-15)
    assert MMS(gamma=2, k=2).u(0.0, 0.0, 0.0) == float(ex["u_gamma2_origin"][0])
    assert MMS(gamma=9, k=9).u(0.0, 0.0, 0.0) == float(ex["u_gamma9_origin"][0])
    assert estimate_rates([1, 1 / 16], [16, 32])[0] == pytest.approx(float(ex["rate_16_32"][0]))
    assert trimmed_average([1, 2, 3]) == float(ex["trimmed_123"][0])
    assert MMS().u(1 / 16, 1 / 16, 0) == pytest.approx(1.0)
    assert MMS().u(0.3, 0.7, T / 4) == pytest.approx(0.0, abs=1e-15)


def test_step_counts_at_N1024():
    """5T at N=1024: 3979 CFD / 4470 MFD steps (SURVEY SA-13, [G16])."""
    assert dt_rate_study(1 / 1024, 0.91, 5 * T)[1] == 3979
    assert dt_rate_study(1 / 1024, 0.81, 5 * T)[1] == 4470


@pytest.mark.parametrize("name,col,printed", [
    ("paper_table3_cfd_rates.txt", 1, 4.02), ("paper_table3_cfd_rates.txt", 2, 2.07),
    ("paper_table3_cfd_rates.txt", 3, 2.02), ("paper_table4_mfd_rates.txt", 1, 3.87),
    ("paper_table4_mfd_rates.txt", 2, 1.99), ("paper_table4_mfd_rates.txt", 3, 1.88)])
def test_trimmed_average_reproduces_tables(name, col, printed):
    rows = read_golden(name)
    rates = [float(r[col]) for r in rows if r[0] != "AVG"]
    avg = [float(r[col]) for r in rows if r[0] == "AVG"][0]
    assert avg == printed
    assert trimmed_average(rates) == pytest.approx(printed, abs=0.01)


def _mms_error(method, n, case, **kw):
    p = mms_problem(method, n, case, **kw)
    U, _, _ = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W,
                         nsteps=p.meta["steps"], **p.oracle_kwargs())
    return interior_error(p, U, p.meta["t_end"])


def test_mfd_rate_near_four_gamma0():
    """MFD, Γ=0, T_sim=5T, cfl 0.81, K=8 on 41->81->161 nodes: rates near 4
    ("convergence rates close to 4"; Table 4 Γ=0)."""
    Ns = [40, 80, 160]
    errs = [_mms_error(MFD, N + 1, MMS(), t_sim=5 * T) for N in Ns]
    r = estimate_rates(errs, Ns)
    assert errs[0] > errs[1] > errs[2]
    assert all(3.3 < x < 5.5 for x in r), r
    assert math.log(errs[0] / errs[2]) / math.log(4) > 3.8


def test_mfd_rate_near_two_gamma2():
    """MFD, Γ=k=2: convergence decays toward second order (Table 4)."""
    Ns = [80, 160]
    errs = [_mms_error(MFD, N + 1, MMS(gamma=2, k=2), t_sim=5 * T) for N in Ns]
    r = estimate_rates(errs, Ns)[0]
    assert 1.4 < r < 2.6, r


def test_cfd_short_horizon_time_order():
    """CFD at t = T/8: the error is dominated by the O(Δt²) CN time error; with
    Δt ∝ h the unnormalized Frobenius error (sum over N² points) falls like
    N^(-1), i.e. second order in the h-weighted L2 norm."""
    Ns = [40, 80, 160]
    errs = [_mms_error(CFD, N + 1, MMS(), t_sim=T / 8) for N in Ns]
    r = estimate_rates(errs, Ns)
    assert errs[0] > errs[1] > errs[2]
    assert all(0.8 < x < 1.3 for x in r), r
