"""A container for one ADI run's inputs (state + source + boundary + tables)."""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np

from .grid import CFD, Grid, interior_shape, shapes


@dataclass
class Problem:
    method: int
    nx: int
    ny: int
    h: float
    dt: float
    c: float
    K: int
    U: np.ndarray
    V: np.ndarray
    W: np.ndarray
    phi: Optional[np.ndarray] = None          # dense source pattern (pressure interior)
    src: Optional[Tuple[int, int]] = None     # point source (ix, iy) in U indices, F = g/h^2
    gf: Optional[np.ndarray] = None           # source time function at half steps
    edges: Optional[Tuple[np.ndarray, ...]] = None   # (y0, y1, x0, x1) boundary pattern
    gb: Optional[np.ndarray] = None           # boundary time function at half steps
    rho: float = 1.0
    meta: dict = field(default_factory=dict)
    # heterogeneous media (NEXT row f3): kappa on the U layout, rho^-1 on the V̄ and
    # W̄ layouts; fp32 arrays (the GPU path's material precision)
    kappa: Optional[np.ndarray] = None
    rinv_v: Optional[np.ndarray] = None
    rinv_w: Optional[np.ndarray] = None

    def oracle_kwargs(self):
        kw = dict(rho=self.rho, phi=self.phi, src=self.src, gf=self.gf, edges=self.edges,
                  gb=self.gb)
        if self.kappa is not None:
            kw.update(kappa=self.kappa, rinv_v=self.rinv_v, rinv_w=self.rinv_w)
        return kw


def random_problem(method: int, n: int, *, seed: int = 0, cfl: float = None, K: int = 8,
                   steps: int = 4, source: bool = True, boundary: bool = True,
                   ny: int = None, media: bool = False) -> Problem:
    """Seeded random state with a random dense source and random boundary data.

    Values are O(1) normal; tables cover ``steps`` steps.  Used for parity
    and invariant tests (no structure assumed by the method).  ``media``: random
    fp32 kappa and rho^-1 fields, uniform in [0.6, 1] (c <= 1, so the homogeneous
    CFL numbers still apply).
    """
    rng = np.random.default_rng(seed)
    if cfl is None:
        cfl = 0.91 if method == CFD else 0.81
    nx, ny = n, (n if ny is None else ny)
    h = 1.0 / (max(nx, ny) - 1)   # one spacing in both directions (the domain may be a rectangle)
    dt = h * cfl
    su, sv, sw = shapes(method, nx, ny)
    U = rng.standard_normal(su)
    V = rng.standard_normal(sv)
    W = rng.standard_normal(sw)
    phi = rng.standard_normal(interior_shape(method, nx, ny)) if source else None
    nt = 2 * steps + 1
    gf = rng.standard_normal(nt) if source else None
    edges = None
    gb = None
    if boundary:
        edges = (rng.standard_normal(su[1]), rng.standard_normal(su[1]),
                 rng.standard_normal(su[0]), rng.standard_normal(su[0]))
        gb = rng.standard_normal(nt)
    med = {}
    if media:
        med = {k: rng.uniform(0.6, 1.0, s_).astype(np.float32)
               for k, s_ in (("kappa", su), ("rinv_v", sv), ("rinv_w", sw))}
    return Problem(method, nx, ny, h, dt, 1.0, K, U, V, W, phi=phi, gf=gf, edges=edges, gb=gb,
                   meta=dict(kind="random", seed=seed, cfl=cfl, steps=steps), **med)
