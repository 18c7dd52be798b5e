"""The parity bar shared by the GPU tests.

Per field, element by element on the same seeded inputs:
* relative L2:   ||a - b||_2 / ||b||_2      <= ``tol``  (north_star: 1e-12);
* relative max:  ||a - b||_inf / ||b||_inf  <= ``maxtol`` (default 10 x tol: 1e-11).

The max-norm bound catches a few wrong points (line ends, segment seams, band
cuts) that a relative L2 over 2.7e8 points would dilute by ~sqrt(N).  Where
``floor`` (the oracle's own relative change under a 1-ulp input perturbation,
per field) is given, both bounds are raised to 10x / 100x of it: a comparison
cannot be better conditioned than the problem.
"""
import numpy as np

TOL = 1e-12
MAXTOL = 1e-11


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def maxrel(a, b):
    mb = np.abs(b).max() if b.size else 0.0
    return float(np.abs(a - b).max() / (mb if mb > 0 else 1.0)) if b.size else 0.0


def check(a, b, tol=TOL, maxtol=MAXTOL, what="", name=""):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, f"{what} {name}: shape {a.shape} != {b.shape}"
    r, m = rel(a, b), maxrel(a, b)
    assert r <= tol, f"{what} {name}: rel L2 {r:.3e} > {tol:.1e}"
    assert m <= maxtol, f"{what} {name}: rel max {m:.3e} > {maxtol:.1e}"


def assert_parity(g, o, tol=TOL, what="", floor=None, maxtol=None):
    for k, (name, a, b) in enumerate(zip("UVW", g, o)):
        lim = tol if floor is None else max(tol, 10 * floor[k])
        mlim = 10 * tol if maxtol is None else maxtol
        if floor is not None:
            mlim = max(mlim, 100 * floor[k])
        check(a, b, lim, mlim, what, name)
