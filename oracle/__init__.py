"""CPU fp64 oracle for the ADI hot path of arXiv:2006.07583 — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_2006_07583_b200``) never imports it; the two share no
code.  The arithmetic lives in ``adi_oracle.c`` (plain C, fp64, no FMA
contraction, OpenMP over independent grid lines); this module only marshals
numpy arrays into it.  See the C file header for the paper passages each
function follows, and DESIGN.md §3-4 for the readings and pins.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

CFD = 0
MFD = 1
_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "adi_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain -O3, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O3", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-Wall", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        D = ctypes.c_double
        I = ctypes.c_int
        P = ctypes.c_void_p
        _lib.or_run_flat.argtypes = [I, I, I, D, D, D, D, I, P, I, I, P, I, P, P, P, P, P, I,
                                     P, P, P, I, I, I, D, I, P, P, P, P, P]
        _lib.or_run_flat.restype = I
        _lib.or_apply_D.argtypes = [I, I, D, P, P]
        _lib.or_apply_Dbar.argtypes = [I, I, D, P, P]
        _lib.or_stage_line.argtypes = [I, I, D, I, D, D, P, P, P, P, D, D, P, P]
        _lib.or_cfd_factors.argtypes = [I, I, P, P]
        _lib.or_tri_factor.argtypes = [I, P, P, P, P, P]
        _lib.or_tri_solve.argtypes = [I, P, P, P, P, P]
        _lib.or_tri_solve.restype = None
        _lib.or_cfd_Qf.argtypes = [I, D, P, P]
        _lib.or_cfd_Qbarf.argtypes = [I, D, P, P]
        _lib.or_mfd_D4f.argtypes = [I, D, P, P]
        _lib.or_mfd_G4f.argtypes = [I, D, P, P]
        for f in (_lib.or_cfd_Qf, _lib.or_cfd_Qbarf, _lib.or_mfd_D4f, _lib.or_mfd_G4f):
            f.restype = None
        _lib.or_num_threads.restype = I
        _lib.or_run_full_flat.argtypes = [I, I, D, D, D, D, I, P, I, I, P, I, P, P, P, I, I, I, I, D]
        _lib.or_run_full_flat.restype = I
        _lib.or_stage_line_full.argtypes = [I, D, I, D, D, P, P, P, P]
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def shapes(method: int, nx: int, ny: int):
    """(U, V̄, W̄) shapes of the state."""
    if method == CFD:
        return (ny, nx), (ny - 2, nx), (ny, nx - 2)
    return (ny + 1, nx + 1), (ny - 1, nx), (ny, nx - 1)


def interior_shape(method: int, nx: int, ny: int):
    return (ny - 2, nx - 2) if method == CFD else (ny - 1, nx - 1)


def run(method, nx, ny, h, dt, c, K, U, V, W, *, rho=1.0, phi=None, src=None, gf=None,
        edges=None, gb=None, m0=0, nsteps=1, nthreads=0, eps=0.0, kmin=6, info=None,
        kappa=None, rinv_v=None, rinv_w=None):
    """Advance copies of (U, V̄, W̄) by ``nsteps`` ADI steps; returns new arrays.

    ``eps`` > 0 applies the stopping rule of Alg. 3/4 (sweeps ``kmin``..K tested,
    test_k = ||U_k - U_{k-1}||_F + ||V_k - V_{k-1}||_F over the stage); ``info``
    (a dict) then receives "k" [nsteps, 2] (chosen sweeps, rows / columns) and
    "tests" [nsteps, 2, K+1].

    ``edges`` = (y0, y1, x0, x1) boundary pattern on the U edges (or None for
    homogeneous Dirichlet); ``gf``/``gb`` are the source / boundary time
    functions sampled at half steps, g[j] = g(j*dt/2) (None means 1).
    ``src`` = (ix, iy) U-array indices of a point source F = g_f/h^2.

    Heterogeneous media (NEXT row f3): ``kappa`` on the U layout
    (interior points used), ``rinv_v`` = rho^-1 on the V̄ layout, ``rinv_w`` on
    the W̄ layout; all three or none (then the scalars c, rho: kappa = rho c^2).
    """
    su, sv, sw = shapes(method, nx, ny)
    U = np.array(U, dtype=np.float64, order="C", copy=True).reshape(su)
    V = np.array(V, dtype=np.float64, order="C", copy=True).reshape(sv)
    W = np.array(W, dtype=np.float64, order="C", copy=True).reshape(sw)
    phi = _f64(phi)
    if phi is not None:
        assert phi.shape == interior_shape(method, nx, ny)
    gf = _f64(gf)
    gb = _f64(gb)
    if edges is None:
        e = [None] * 4
    else:
        e = [_f64(x) for x in edges]
        assert e[0].size == su[1] and e[1].size == su[1] and e[2].size == su[0] and e[3].size == su[0]
    med = [kappa, rinv_v, rinv_w]
    if any(m is not None for m in med):
        assert all(m is not None for m in med), "kappa, rinv_v, rinv_w: all or none"
        med = [_f64(m) for m in med]
        assert med[0].shape == su and med[1].shape == sv and med[2].shape == sw
    ix, iy = (-1, -1) if src is None else src
    kch = np.zeros((max(nsteps, 1), 2), dtype=np.int32)
    tests = np.zeros((max(nsteps, 1), 2, K + 1))
    rc = lib().or_run_flat(method, nx, ny, h, dt, c, rho, K, _p(phi), ix, iy, _p(gf),
                           0 if gf is None else gf.size, _p(e[0]), _p(e[1]), _p(e[2]), _p(e[3]),
                           _p(gb), 0 if gb is None else gb.size, _p(U), _p(V), _p(W), m0, nsteps,
                           nthreads, float(eps), int(kmin), _p(kch), _p(tests), _p(med[0]),
                           _p(med[1]), _p(med[2]))
    if rc != 0:
        raise RuntimeError(f"oracle or_run failed: {rc}")
    if info is not None:
        info["k"] = kch[:nsteps]
        info["tests"] = tests[:nsteps]
    return U, V, W


def apply_D(method, n, h, ub):
    """D = P^-1 Q (CFD, n+1 -> n+1) or G4 (MFD, n+2 -> n+1) on one line."""
    ub = _f64(ub)
    out = np.zeros(n + 1)
    assert lib().or_apply_D(method, n, h, _p(ub), _p(out)) == 0
    return out


def apply_Dbar(method, n, h, v):
    """D̄ = P̄^-1 Q̄ (CFD, n+1 -> n-1) or D4 (MFD, n+1 -> n) on one line."""
    v = _f64(v)
    out = np.zeros(n - 1 if method == CFD else n)
    assert lib().or_apply_Dbar(method, n, h, _p(v), _p(out)) == 0
    return out


def stage_line(method, n, h, K, alpha, beta, s, v0, gL, gR):
    """One stage on one line; ``alpha`` / ``beta`` scalars or per-point arrays (f3)."""
    s = _f64(s)
    v0 = _f64(v0)
    u = np.zeros(n - 1 if method == CFD else n)
    v = np.zeros(n + 1)
    av = None if np.isscalar(alpha) else _f64(alpha)
    bv = None if np.isscalar(beta) else _f64(beta)
    assert av is None or av.size == u.size
    assert bv is None or bv.size == v.size
    a0 = float(alpha) if av is None else 0.0
    b0 = float(beta) if bv is None else 0.0
    assert lib().or_stage_line(method, n, h, K, a0, b0, _p(av), _p(bv), _p(s), _p(v0), gL, gR,
                               _p(u), _p(v)) == 0
    return u, v


def cfd_factors(n, which):
    """LU multipliers l and pivots d of P (which=0, size n+1) or P̄ (which=1, n-1)."""
    m = n + 1 if which == 0 else n - 1
    l = np.zeros(m)
    d = np.zeros(m)
    assert lib().or_cfd_factors(n, which, _p(l), _p(d)) == 0
    return l, d


def tri_factor(a, b, c):
    a, b, c = _f64(a), _f64(b), _f64(c)
    n = b.size
    l = np.zeros(n)
    d = np.zeros(n)
    rc = lib().or_tri_factor(n, _p(a), _p(b), _p(c), _p(l), _p(d))
    return rc, l, d


def tri_solve(l, d, c, r):
    l, d, c, r = _f64(l), _f64(d), _f64(c), _f64(r)
    x = np.zeros(r.size)
    lib().or_tri_solve(r.size, _p(l), _p(d), _p(c), _p(r), _p(x))
    return x


def raw_operator(name, n, h, f):
    """The raw banded products Q f, Q̄ f, D4 f, G4 f (no solve)."""
    f = _f64(f)
    size = {"Q": n + 1, "Qbar": n - 1, "D4": n, "G4": n + 1}[name]
    out = np.zeros(size)
    fn = {"Q": lib().or_cfd_Qf, "Qbar": lib().or_cfd_Qbarf, "D4": lib().or_mfd_D4f,
          "G4": lib().or_mfd_G4f}[name]
    fn(n, h, _p(f), _p(out))
    return out


def num_threads() -> int:
    return lib().or_num_threads()


def run_full(nx, ny, h, dt, c, K, U, V, W, *, rho=1.0, phi=None, src=None, gf=None, m0=0, nsteps=1,
             nthreads=0, nb=0, a=0.015):
    """NEXT row f4: the full-matrix CFD variant (readings F1-F2 in
    adi_oracle.c): U, V, W are all ny x nx (every node unknown, no Dirichlet data),
    every derivative is the full D = P^-1 Q, and after each step all fields are
    multiplied by the Cerjan taper G(x) G(y) of width ``nb`` (0: none) and rate ``a``.
    ``phi``: dense source on all nodes (ny x nx); ``src`` = (ix, iy) node of a point
    source F = g_f / h^2."""
    U, V, W = (np.array(x, dtype=np.float64, order="C", copy=True).reshape(ny, nx) for x in (U, V, W))
    phi = _f64(phi)
    if phi is not None:
        assert phi.shape == (ny, nx)
    gf = _f64(gf)
    ix, iy = (-1, -1) if src is None else src
    rc = lib().or_run_full_flat(nx, ny, h, dt, c, rho, K, _p(phi), ix, iy, _p(gf), 0 if gf is None else gf.size,
                                _p(U), _p(V), _p(W), m0, nsteps, nthreads, int(nb), float(a))
    if rc != 0:
        raise RuntimeError(f"oracle or_run_full failed: {rc}")
    return U, V, W


def stage_line_full(n, h, K, alpha, beta, s, v0):
    """One full-variant stage on one line (f4, reading F1): K sweeps of
    u = s - alpha D v, v = v0 - beta D u with the full D = P^-1 Q (n+1 nodes)."""
    s, v0 = _f64(s), _f64(v0)
    u, v = np.zeros(n + 1), np.zeros(n + 1)
    assert lib().or_stage_line_full(n, h, K, alpha, beta, _p(s), _p(v0), _p(u), _p(v)) == 0
    return u, v
