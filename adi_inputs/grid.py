"""Grid layouts of the two methods.

Row index = y, column index = x.  ``nx``/``ny`` are node counts per direction
(N = n - 1 cells, h = 1/N on the unit square).

* CFD (nodal): U ny x nx incl. boundary; V̄ (ny-2) x nx; W̄ ny x (nx-2).
* MFD (staggered): U (ny+1) x (nx+1) on X_cb x Y_cb; V̄ (ny-1) x nx
  (x nodes, y centres); W̄ ny x (nx-1) (y nodes, x centres).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

CFD = 0
MFD = 1
CFD_FULL = 2   # the full-matrix CFD variant (NEXT row f4): every node is state


def shapes(method: int, nx: int, ny: int):
    if method == CFD_FULL:
        return (ny, nx), (ny, nx), (ny, nx)
    if method == CFD:
        return (ny, nx), (ny - 2, nx), (ny, nx - 2)
    return (ny + 1, nx + 1), (ny - 1, nx), (ny, nx - 1)


def interior_shape(method: int, nx: int, ny: int):
    if method == CFD_FULL:
        return (ny, nx)
    return (ny - 2, nx - 2) if method == CFD else (ny - 1, nx - 1)


def nodes(n_nodes: int) -> np.ndarray:
    """X_n = (x_0 .. x_N), x_i = i h."""
    N = n_nodes - 1
    return np.arange(n_nodes, dtype=np.float64) / N


def cb_points(n_nodes: int) -> np.ndarray:
    """X_cb = (0, x_1/2, ..., x_{N-1/2}, 1)."""
    N = n_nodes - 1
    x = np.empty(N + 2)
    x[0] = 0.0
    x[1:N + 1] = (np.arange(N, dtype=np.float64) + 0.5) / N
    x[N + 1] = 1.0
    return x


@dataclass(frozen=True)
class Grid:
    method: int
    nx: int
    ny: int

    @property
    def h(self) -> float:
        assert self.nx == self.ny, "the paper's grids are square (h = 1/N)"
        return 1.0 / (self.nx - 1)

    def u_xy(self):
        """Coordinates of the U array (incl. boundary)."""
        if self.method == CFD:
            return nodes(self.nx), nodes(self.ny)
        return cb_points(self.nx), cb_points(self.ny)

    def v_xy(self):
        """Coordinates of V̄: x at nodes, y at interior pressure rows."""
        xu, yu = self.u_xy()
        return nodes(self.nx), yu[1:-1]

    def w_xy(self):
        """Coordinates of W̄: x at interior pressure columns, y at nodes."""
        xu, yu = self.u_xy()
        return xu[1:-1], nodes(self.ny)

    def interior_xy(self):
        xu, yu = self.u_xy()
        return xu[1:-1], yu[1:-1]


def dt_for_cfl(h: float, cfl: float, c: float = 1.0) -> float:
    """Δt = h c^{-1} cfl (Alg. 1 line 2)."""
    return h * cfl / c


def dt_rate_study(h: float, cfl: float, t_sim: float, c: float = 1.0):
    """Δt that lands exactly on T_sim: T_sim / ceil(T_sim c / (cfl h)) [G16]."""
    steps = int(math.ceil(t_sim * c / (cfl * h) - 1e-12))
    return t_sim / steps, steps
