"""A manufactured solution in a HETEROGENEOUS medium (NEXT row f3).

Eq. 1 with fields K = kappa(x,y), R = rho^-1(x,y), written as
u_t + kappa (v_x + w_y) = f, v_t = -R u_x, w_t = -R u_y (the homogeneous MMS
of ``mms`` with rho v_t = -u_x).  With the spatial factor S of eq. 11
(Γ = 0: S = sin(ax) sin(ay)):

    u = S cos ωt
    v = -R S_x sin ωt / ω,   w = -R S_y sin ωt / ω
    f = -sin ωt [ω S + (kappa/ω) (∂x(R S_x) + ∂y(R S_y))]

so the source is still separable, F = φ(x,y) g_f(t) with g_f = sin ωt, and the
Dirichlet data S|∂Ω cos ωt.  The medium: kappa = k0 (1 + ak sin(2πx + 0.3)
cos(2πy)), R = r0 (1 + ar cos(2πx) sin(2πy + 0.7)), smooth, positive.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .grid import Grid, dt_rate_study, shapes
from .problem import Problem


@dataclass(frozen=True)
class Medium:
    k0: float = 1.0
    ak: float = 0.25
    r0: float = 1.0
    ar: float = 0.25

    def kappa(self, x, y):
        return self.k0 * (1.0 + self.ak * np.sin(2 * math.pi * x + 0.3) * np.cos(2 * math.pi * y))

    def R(self, x, y):
        return self.r0 * (1.0 + self.ar * np.cos(2 * math.pi * x) * np.sin(2 * math.pi * y + 0.7))

    def R_x(self, x, y):
        return -self.r0 * self.ar * 2 * math.pi * np.sin(2 * math.pi * x) * np.sin(2 * math.pi * y + 0.7)

    def R_y(self, x, y):
        return self.r0 * self.ar * 2 * math.pi * np.cos(2 * math.pi * x) * np.cos(2 * math.pi * y + 0.7)

    @property
    def c_max(self) -> float:
        return math.sqrt(self.k0 * (1 + self.ak) * self.r0 * (1 + self.ar))


@dataclass(frozen=True)
class MediumMMS:
    lam: float = 0.25
    T: float = 1.0 / math.sqrt(2.0)
    medium: Medium = Medium()

    @property
    def a(self):
        return 2.0 * math.pi / self.lam

    @property
    def omega(self):
        return 2.0 * math.pi / self.T

    def S(self, x, y):
        return np.sin(self.a * x) * np.sin(self.a * y)

    def S_x(self, x, y):
        return self.a * np.cos(self.a * x) * np.sin(self.a * y)

    def S_y(self, x, y):
        return self.S_x(y, x)

    def div_R_grad_S(self, x, y):
        m, a = self.medium, self.a
        S_xx = -a * a * self.S(x, y)
        return m.R_x(x, y) * self.S_x(x, y) + m.R_y(x, y) * self.S_y(x, y) + m.R(x, y) * 2.0 * S_xx

    def u(self, x, y, t):
        return self.S(x, y) * math.cos(self.omega * t)

    def v(self, x, y, t):
        return -self.medium.R(x, y) * self.S_x(x, y) * math.sin(self.omega * t) / self.omega

    def w(self, x, y, t):
        return -self.medium.R(x, y) * self.S_y(x, y) * math.sin(self.omega * t) / self.omega

    def phi(self, x, y):
        w = self.omega
        return -(w * self.S(x, y) + (self.medium.kappa(x, y) / w) * self.div_R_grad_S(x, y))


def medium_mms_problem(method: int, n: int, case: MediumMMS = MediumMMS(), *, cfl: float = 0.81,
                       K: int = 8, t_sim: float = None, steps: int = None, f32: bool = False) -> Problem:
    """The medium MMS on an n x n node grid; Δt from cfl and the medium's c_max.

    ``f32``: the material fields rounded to fp32 (the GPU path's input type); the
    exact solution then belongs to a medium perturbed by ~1e-8 (below every error
    measured here)."""
    g = Grid(method, n, n)
    h = g.h
    c = case.medium.c_max
    if t_sim is not None:
        dt, steps = dt_rate_study(h, cfl, t_sim, c)
    else:
        dt = cfl * h / c
    assert steps is not None
    xu, yu = g.u_xy()
    xv, yv = g.v_xy()
    xw, yw = g.w_xy()
    su, sv, sw = shapes(method, n, n)
    U = case.S(xu[None, :], yu[:, None]) * 1.0
    V = case.v(xv[None, :], yv[:, None], 0.0) * np.ones(sv)
    W = case.w(xw[None, :], yw[:, None], 0.0) * np.ones(sw)
    xi, yi = g.interior_xy()
    phi = case.phi(xi[None, :], yi[:, None])
    edges = (case.S(xu, 0.0 * xu), case.S(xu, 0.0 * xu + 1.0),
             case.S(0.0 * yu, yu), case.S(0.0 * yu + 1.0, yu))
    tt = np.arange(2 * steps + 1, dtype=np.float64) * (dt / 2.0)
    gf = np.sin(case.omega * tt)
    gb = np.cos(case.omega * tt)
    m = case.medium
    kap = m.kappa(xu[None, :], yu[:, None]) * np.ones(su)
    rv = m.R(xv[None, :], yv[:, None]) * np.ones(sv)
    rw = m.R(xw[None, :], yw[:, None]) * np.ones(sw)
    if f32:
        kap, rv, rw = (a.astype(np.float32) for a in (kap, rv, rw))
    return Problem(method, n, n, h, dt, c, K, U, V, W, phi=phi, gf=gf, edges=edges, gb=gb,
                   kappa=kap, rinv_v=rv, rinv_w=rw,
                   meta=dict(kind="medium_mms", case=case, steps=steps, cfl=cfl, t_end=steps * dt))


def medium_error(p: Problem, U: np.ndarray, t: float) -> float:
    """Unnormalized Frobenius error of interior U at time t [G17]."""
    g = Grid(p.method, p.nx, p.ny)
    xu, yu = g.u_xy()
    Ue = p.meta["case"].u(xu[None, :], yu[:, None], t)
    return float(np.linalg.norm((U - Ue)[1:-1, 1:-1]))
