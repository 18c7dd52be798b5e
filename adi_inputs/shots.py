"""Ricker point-source shots (config 5 of BASELINE.json).

r(t) = (1 - 2π² f0² (t-t0)²) exp(-π² f0² (t-t0)²), f0 = 100 Hz, t0 = 0.015 s;
shot s at cell (0.1 + 0.8 s/63, 0.05); zero initial fields; homogeneous
Dirichlet (free surface) on all edges; F = r(t)/h² at the source cell.
"""
from __future__ import annotations

import math

import numpy as np

from .grid import MFD, Grid, interior_shape, shapes
from .problem import Problem


def ricker(t, f0: float = 100.0, t0: float = 0.015):
    a = (math.pi * f0 * (np.asarray(t) - t0)) ** 2
    return (1.0 - 2.0 * a) * np.exp(-a)


def shot_position(s: int, nshots: int = 64):
    return 0.1 + 0.8 * s / max(nshots - 1, 1), 0.05


def ricker_problem(n: int, shot: int = 0, *, method: int = MFD, nshots: int = 64, cfl: float = 0.81,
                   steps: int = 100, K: int = 8, f0: float = 100.0, t0: float = 0.015) -> Problem:
    g = Grid(method, n, n)
    h = g.h
    dt = h * cfl
    su, sv, sw = shapes(method, n, n)
    xs, ys = shot_position(shot, nshots)
    xu, yu = g.u_xy()
    ix = int(np.argmin(np.abs(xu[1:-1] - xs))) + 1
    iy = int(np.argmin(np.abs(yu[1:-1] - ys))) + 1
    tt = np.arange(2 * steps + 1, dtype=np.float64) * (dt / 2.0)
    return Problem(method, n, n, h, dt, 1.0, K, np.zeros(su), np.zeros(sv), np.zeros(sw),
                   src=(ix, iy), gf=ricker(tt, f0, t0), edges=None, gb=None,
                   meta=dict(kind="ricker", shot=shot, steps=steps, cfl=cfl, f0=f0, t0=t0))
