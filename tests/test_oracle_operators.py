"""Pins for the oracle's operators (Appendix A/B) and its tridiagonal LU.

Every check here is fixed by something other than the oracle itself:
the printed rows of the paper (tests/golden), exact polynomial moments
(the operators are 4th-order accurate: PAPER.md:554, 618), exact Gaussian
elimination in rational arithmetic, numpy's dense solver, and reflection
symmetry of the continuous derivative.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import CFD, MFD
from conftest import read_golden


def _golden_rows():
    rows = {}
    for r in read_golden("appendix_operators.txt"):
        name, kind, off = r[0], r[1], int(r[2])
        coef = [Fraction(x) for x in r[3:]]
        rows[(name, kind)] = (off, coef)
    return rows


def _dense_raw(name, n):
    """The raw banded product matrix (no solve), read column by column from the oracle."""
    cols = {"Q": n + 1, "Qbar": n + 1, "D4": n + 1, "G4": n + 2}[name]
    mats = [oracle.raw_operator(name, n, 1.0, np.eye(cols)[j]) for j in range(cols)]
    return np.stack(mats, axis=1)


@pytest.mark.parametrize("n", [8, 9, 16, 23])
def test_printed_rows_Q_Qbar(n):
    """Q4, Q̄4 rows equal the printed rationals (eq. 13, 15)."""
    g = _golden_rows()
    for name in ("Q", "Qbar"):
        M = _dense_raw(name, n)
        off, c = g[(name, "first")]
        np.testing.assert_array_equal(M[0, off:off + len(c)], [float(x) for x in c])
        assert np.all(M[0, off + len(c):] == 0)
        off, c = g[(name, "interior")]
        for r in range(1, M.shape[0] - 1):
            start = r - 1 if name == "Q" else r
            np.testing.assert_array_equal(M[r, start:start + 3], [float(x) for x in c])
            assert np.count_nonzero(M[r]) == 2
        off, c = g[(name, "last")]
        np.testing.assert_array_equal(M[-1, off:], [float(x) for x in c])
        assert np.all(M[-1, :off] == 0)


@pytest.mark.parametrize("n", [8, 11, 16])
def test_printed_rows_D4_G4(n):
    """D4, G4 rows equal the printed rationals; bottom rows are the top rows
    reversed and negated (Appendix B)."""
    g = _golden_rows()
    D4 = _dense_raw("D4", n)
    G4 = _dense_raw("G4", n)
    f = lambda c: np.array([float(x) for x in c])
    _, c0 = g[("D4", "first")]
    np.testing.assert_allclose(D4[0, :6], f(c0), rtol=0, atol=1e-15)
    np.testing.assert_allclose(D4[-1, -6:], -f(c0)[::-1], rtol=0, atol=1e-15)
    _, ci = g[("D4", "interior")]
    for r in range(1, n - 1):
        np.testing.assert_allclose(D4[r, r - 1:r + 3], f(ci), rtol=0, atol=1e-15)
    _, g0 = g[("G4", "first")]
    _, g1 = g[("G4", "second")]
    np.testing.assert_allclose(G4[0, :6], f(g0), rtol=0, atol=1e-15)
    np.testing.assert_allclose(G4[1, :5], f(g1), rtol=0, atol=1e-15)
    np.testing.assert_allclose(G4[-1, -6:], -f(g0)[::-1], rtol=0, atol=1e-15)
    np.testing.assert_allclose(G4[-2, -5:], -f(g1)[::-1], rtol=0, atol=1e-15)
    for i in range(2, n - 1):
        np.testing.assert_allclose(G4[i, i - 1:i + 3], f(ci), rtol=0, atol=1e-15)


def _points(method, n, which):
    """Sample positions on [0,1] for the operator inputs/outputs (h = 1/n)."""
    nodes = np.arange(n + 1) / n
    if which == "nodes":
        return nodes
    if which == "inodes":
        return nodes[1:-1]
    if which == "centres":
        return (np.arange(n) + 0.5) / n
    if which == "cb":
        return np.concatenate([[0.0], (np.arange(n) + 0.5) / n, [1.0]])
    raise ValueError


CASES = [  # (method, op, input points, output points)
    (CFD, "D", "nodes", "nodes"),
    (CFD, "Dbar", "nodes", "inodes"),
    (MFD, "D", "cb", "nodes"),        # G4
    (MFD, "Dbar", "nodes", "centres"),  # D4
]


@pytest.mark.parametrize("method,op,pin,pout", CASES)
@pytest.mark.parametrize("n", [8, 16, 32])
def test_polynomial_exactness(method, op, pin, pout, n):
    """4th-order operators differentiate x^p exactly for p <= 4 at every output
    point, closures included ("fourth order accurate"; 618)."""
    h = 1.0 / n
    xi = _points(method, n, pin)
    xo = _points(method, n, pout)
    for p in range(0, 5):
        f = xi ** p
        d = oracle.apply_D(method, n, h, f) if op == "D" else oracle.apply_Dbar(method, n, h, f)
        exact = p * xo ** (p - 1) if p > 0 else 0 * xo
        np.testing.assert_allclose(d, exact, rtol=0, atol=1e-10 * n)


@pytest.mark.parametrize("method,op,pin,pout", CASES)
def test_not_fifth_order(method, op, pin, pout):
    """Sensitivity check: x^5 is NOT differentiated exactly (the pins above
    would also pass a wrong operator only if it were exact to degree 5)."""
    n = 16
    h = 1.0 / n
    xi = _points(method, n, pin)
    xo = _points(method, n, pout)
    d = oracle.apply_D(method, n, h, xi ** 5) if op == "D" else oracle.apply_Dbar(method, n, h, xi ** 5)
    assert np.max(np.abs(d - 5 * xo ** 4)) > 1e-8


@pytest.mark.parametrize("method,op,pin,pout", CASES)
def test_reflection_antisymmetry(method, op, pin, pout):
    """d/dx anticommutes with x -> 1-x; the operators are centro-antisymmetric."""
    n = 19
    h = 1.0 / n
    rng = np.random.default_rng(3)
    f = rng.standard_normal(_points(method, n, pin).size)
    A = oracle.apply_D if op == "D" else oracle.apply_Dbar
    np.testing.assert_allclose(A(method, n, h, f[::-1]), -A(method, n, h, f)[::-1], rtol=0,
                               atol=1e-12 * n)


@pytest.mark.parametrize("n", [16, 64])
def test_reduced_operator_is_interior_of_full(n):
    """P̄^-1 Q̄ equals the interior rows of P^-1 Q (App. A: the reduced formula
    at x_1 is a combination of the original formulas at x_0 and x_1,
    PAPER.md:580; SURVEY SA-2)."""
    rng = np.random.default_rng(n)
    f = rng.standard_normal(n + 1)
    full = oracle.apply_D(CFD, n, 1.0 / n, f)
    red = oracle.apply_Dbar(CFD, n, 1.0 / n, f)
    np.testing.assert_allclose(red, full[1:n], rtol=0, atol=1e-12 * n * np.abs(full).max())


def test_lu_pivots_spec_example():
    """(1,4,1), n=5 -> pivots 4, 15/4, 56/15, 209/56, 780/209."""
    row = read_golden("spec_examples.txt")
    piv = [float(Fraction(x)) for x in dict((r[0], r[1:]) for r in row)["pivots_141_n5"]]
    rc, l, d = oracle.tri_factor(np.r_[0.0, np.ones(4)], 4.0 * np.ones(5), np.r_[np.ones(4), 0.0])
    assert rc == 0
    np.testing.assert_allclose(d, piv, rtol=1e-15)


def _exact_pivots(a, b, c):
    """Gaussian elimination without pivoting in exact rationals (independent of Thomas)."""
    n = len(b)
    M = [[Fraction(0)] * n for _ in range(n)]
    for i in range(n):
        M[i][i] = Fraction(b[i])
        if i > 0:
            M[i][i - 1] = Fraction(a[i])
        if i < n - 1:
            M[i][i + 1] = Fraction(c[i])
    piv = []
    for k in range(n):
        piv.append(M[k][k])
        for i in range(k + 1, n):
            if M[i][k] != 0:
                f = M[i][k] / M[k][k]
                for j in range(k, n):
                    M[i][j] -= f * M[k][j]
    return piv


@pytest.mark.parametrize("n", [8, 13])
def test_cfd_pivots_exact(n):
    """LU pivots of P4 and P̄4 match exact elimination of the printed matrices
    (eq. 12, 14); no zero pivot although P is not diagonally dominant."""
    g = _golden_rows()
    for which, name, size in ((0, "P", n + 1), (1, "Pbar", n - 1)):
        first = [float(x) for x in g[(name, "first")][1]]
        last = [float(x) for x in g[(name, "last")][1]]
        a = np.r_[0.0, np.ones(size - 1)]
        b = 4.0 * np.ones(size)
        c = np.r_[np.ones(size - 1), 0.0]
        b[0], c[0] = first
        a[-1], b[-1] = last
        piv = [float(x) for x in _exact_pivots(a, b, c)]
        l, d = oracle.cfd_factors(n, which)
        np.testing.assert_allclose(d, piv, rtol=1e-14)
        assert np.all(d != 0)
    l, d = oracle.cfd_factors(8, 0)
    np.testing.assert_allclose(d[:4], [6, 1, 3, 11 / 3], rtol=1e-15)
    assert abs(d[-1] - 1.1769) < 1e-4


@pytest.mark.parametrize("n", [8, 33, 100])
def test_thomas_vs_dense_solve(n):
    rng = np.random.default_rng(n)
    a = np.r_[0.0, rng.uniform(0.5, 1.5, n - 1)]
    c = np.r_[rng.uniform(0.5, 1.5, n - 1), 0.0]
    b = 4.0 + rng.uniform(0, 1, n)
    r = rng.standard_normal(n)
    rc, l, d = oracle.tri_factor(a, b, c)
    assert rc == 0
    x = oracle.tri_solve(l, d, c, r)
    T = np.diag(b) + np.diag(a[1:], -1) + np.diag(c[:-1], 1)
    np.testing.assert_allclose(x, np.linalg.solve(T, r), rtol=1e-13, atol=1e-13)


def test_zero_pivot_detected():
    rc, _, _ = oracle.tri_factor(np.array([0.0, 1.0]), np.array([1.0, 1.0]), np.array([1.0, 0.0]))
    assert rc == -4


@pytest.mark.parametrize("method,op,pin,pout", CASES)
def test_observed_order_sine(method, op, pin, pout):
    """Richardson order on sin(2πx) between N=32 and 64 is ~4."""
    errs = []
    for n in (32, 64):
        xi = _points(method, n, pin)
        xo = _points(method, n, pout)
        A = oracle.apply_D if op == "D" else oracle.apply_Dbar
        d = A(method, n, 1.0 / n, np.sin(2 * np.pi * xi))
        errs.append(np.max(np.abs(d - 2 * np.pi * np.cos(2 * np.pi * xo))))
    assert np.log2(errs[0] / errs[1]) > 3.7
