"""Exact harmonic solution of eq. 11 and its MMS fields.

The paper gives only u.  With S(x,y) = Γ(x^k - (1-x)^k + y^k - (1-y)^k)
+ sin(a x) sin(a y), a = 2π/λ, ω = 2π/T:

    u = S cos ωt
    v = -S_x sin ωt / (ρ ω),   w = -S_y sin ωt / (ρ ω)        (ρ v_t = -u_x)
    f = u_t + κ (v_x + w_y) = -sin ωt [ω S + (κ/(ρ ω)) (S_xx + S_yy)]

so F = φ(x,y) g_f(t) with φ = -[ω S + (κ/(ρω)) ΔS], g_f = sin ωt, and the
Dirichlet data u|∂Ω = S|∂Ω · cos ωt (separable: edges × g_b).  Defaults
λ = 1/4, T = 1/√2, c = 1 (κ = ρ = 1) per PAPER.md:407.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .grid import CFD, Grid, dt_for_cfl, dt_rate_study, shapes
from .problem import Problem


@dataclass(frozen=True)
class MMS:
    gamma: float = 0.0
    k: int = 1
    lam: float = 0.25
    T: float = 1.0 / math.sqrt(2.0)
    kappa: float = 1.0
    rho: float = 1.0

    @property
    def a(self) -> float:
        return 2.0 * math.pi / self.lam

    @property
    def omega(self) -> float:
        return 2.0 * math.pi / self.T

    # spatial factor and derivatives
    def S(self, x, y):
        G, k, a = self.gamma, self.k, self.a
        return G * (x**k - (1 - x)**k + y**k - (1 - y)**k) + np.sin(a * x) * np.sin(a * y)

    def S_x(self, x, y):
        G, k, a = self.gamma, self.k, self.a
        return G * k * (x**(k - 1) + (1 - x)**(k - 1)) + a * np.cos(a * x) * np.sin(a * y)

    def S_y(self, x, y):
        return self.S_x(y, x)

    def lap_S(self, x, y):
        G, k, a = self.gamma, self.k, self.a
        if k >= 2:
            pxx = G * k * (k - 1) * (x**(k - 2) - (1 - x)**(k - 2))
            pyy = G * k * (k - 1) * (y**(k - 2) - (1 - y)**(k - 2))
        else:
            pxx = pyy = 0.0 * x
        return pxx + pyy - 2.0 * a * a * np.sin(a * x) * np.sin(a * y)

    # fields of eq. 1
    def u(self, x, y, t):
        return self.S(x, y) * math.cos(self.omega * t)

    def v(self, x, y, t):
        return -self.S_x(x, y) * math.sin(self.omega * t) / (self.rho * self.omega)

    def w(self, x, y, t):
        return -self.S_y(x, y) * math.sin(self.omega * t) / (self.rho * self.omega)

    def phi(self, x, y):
        w = self.omega
        return -(w * self.S(x, y) + (self.kappa / (self.rho * w)) * self.lap_S(x, y))

    def f(self, x, y, t):
        return self.phi(x, y) * math.sin(self.omega * t)

    @property
    def c(self) -> float:
        return math.sqrt(self.kappa / self.rho)


def mms_problem(method: int, n: int, case: MMS = MMS(), *, cfl: float = None, K: int = 8,
                steps: int = None, t_sim: float = None, dt: float = None) -> Problem:
    """Sample the MMS case on an n x n node grid (N = n-1 cells).

    Either ``t_sim`` (Δt rounded to land on it, [G16]) or ``steps`` with
    Δt = cfl h / c (config 1) or an explicit ``dt``.
    """
    if cfl is None:
        cfl = 0.91 if method == CFD else 0.81
    g = Grid(method, n, n)
    h = g.h
    if t_sim is not None:
        dt, steps = dt_rate_study(h, cfl, t_sim, case.c)
    elif dt is None:
        dt = dt_for_cfl(h, cfl, case.c)
    assert steps is not None
    xu, yu = g.u_xy()
    U = case.S(xu[None, :], yu[:, None]) * 1.0
    su, sv, sw = shapes(method, n, n)
    V = np.zeros(sv)
    W = np.zeros(sw)
    xi, yi = g.interior_xy()
    phi = case.phi(xi[None, :], yi[:, None])
    edges = (case.S(xu, 0.0 * xu), case.S(xu, 0.0 * xu + 1.0),
             case.S(0.0 * yu, yu), case.S(0.0 * yu + 1.0, yu))
    j = np.arange(2 * steps + 1, dtype=np.float64)
    tt = j * (dt / 2.0)
    gf = np.sin(case.omega * tt)
    gb = np.cos(case.omega * tt)
    return Problem(method, n, n, h, dt, case.c, K, U, V, W, phi=phi, gf=gf, edges=edges, gb=gb,
                   rho=case.rho, meta=dict(kind="mms", case=case, steps=steps, cfl=cfl,
                                           t_end=steps * dt))


def exact_fields(p: Problem, t: float):
    """Exact (U, V̄, W̄) of the MMS case at time t on the problem's layout."""
    case = p.meta["case"]
    g = Grid(p.method, p.nx, p.ny)
    xu, yu = g.u_xy()
    xv, yv = g.v_xy()
    xw, yw = g.w_xy()
    U = case.u(xu[None, :], yu[:, None], t)
    V = case.v(xv[None, :], yv[:, None], t)
    W = case.w(xw[None, :], yw[:, None], t)
    return U, V, W


def interior_error(p: Problem, U: np.ndarray, t: float) -> float:
    """Unnormalized Frobenius error of interior U at time t [G17]."""
    Ue, _, _ = exact_fields(p, t)
    return float(np.linalg.norm((U - Ue)[1:-1, 1:-1]))
