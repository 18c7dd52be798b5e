"""GPU parity of the heterogeneous-media path (adi_set_media)
against the oracle, through the C-ABI: relative L2 <= 1e-12 per field on seeded
random fp32 media (kappa, rho^-1 uniform in [0.6, 1]), over the generic tiles
(short lines), the lean tiles with line ends (1601^2), rectangles, batches,
point sources and the medium MMS (adi_inputs.media); plus the reductions
(constant media == the scalar kernels) and the API's error paths."""
import math

import numpy as np
import pytest

import oracle
from adi_inputs import CFD, MFD, random_problem
from adi_inputs.media import MediumMMS, medium_error, medium_mms_problem

from parity import assert_parity, rel  # noqa: E402,F401  (rel L2 + rel max)

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module")
def adi():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2006_07583_b200 as m
    m.lib()
    return m


def run_oracle(p, nsteps):
    return oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=nsteps,
                      **p.oracle_kwargs())


def run_gpu(adi, p, nsteps, split=None):
    s = adi.AdiSolver.from_problem(p)
    for k in (split or [nsteps]):
        s.step(k)
    out = s.get_fields()
    s.close()
    return out


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n,steps", [(21, 4), (41, 3), (333, 2)])
def test_media_parity_generic_tiles(adi, method, n, steps):
    p = random_problem(method, n, seed=100 + n, steps=steps, media=True)
    assert_parity(run_gpu(adi, p, steps), run_oracle(p, steps), what=f"media {n}")


@pytest.mark.parametrize("method", [CFD, MFD])
def test_media_parity_lean_tiles(adi, method):
    p = random_problem(method, 1601, seed=7, steps=2, media=True)
    assert_parity(run_gpu(adi, p, 2, split=[1, 1]), run_oracle(p, 2), what="media 1601")


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("nx,ny", [(77, 2100), (2101, 1602)])
def test_media_parity_rectangles(adi, method, nx, ny):
    p = random_problem(method, nx, ny=ny, seed=nx, steps=2, media=True)
    assert_parity(run_gpu(adi, p, 2), run_oracle(p, 2), what=f"media {nx}x{ny}")


@pytest.mark.parametrize("method", [CFD, MFD])
def test_media_parity_batch(adi, method):
    """A batch of 2 grids sharing one medium, source and boundary (lean tiles)."""
    n, B, steps = 1601, 2, 2
    ps = [random_problem(method, n, seed=60 + b, steps=steps, media=True) for b in range(B)]
    p0 = ps[0]
    s = adi.AdiSolver(n, n, p0.h, p0.dt, p0.c, method, batch=B, K=p0.K)
    s.set_fields(np.stack([p.U for p in ps]), np.stack([p.V for p in ps]), np.stack([p.W for p in ps]))
    s.set_source(p0.phi, None, p0.gf)
    s.set_boundary(p0.edges, p0.gb)
    s.set_media(p0.kappa, p0.rinv_v, p0.rinv_w)
    s.step(steps)
    g = s.get_fields()
    s.close()
    for b, p in enumerate(ps):
        o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=steps,
                       **{**p0.oracle_kwargs(), "rho": p.rho})
        assert_parity([x[b] for x in g], o, what=f"media batch member {b}")


@pytest.mark.parametrize("method", [CFD, MFD])
def test_media_point_source(adi, method):
    p = random_problem(method, 1601, seed=9, steps=3, media=True, source=False)
    p.src = (700, 901)
    p.gf = np.random.default_rng(1).standard_normal(7)
    assert_parity(run_gpu(adi, p, 3), run_oracle(p, 3), what="media point source")


@pytest.mark.parametrize("method", [CFD, MFD])
def test_constant_media_match_scalar_kernels(adi, method):
    """kappa = rho^-1 = 1 through the media kernels == the scalar kernels (to rounding)."""
    p = random_problem(method, 1601, seed=5, steps=2)
    a = run_gpu(adi, p, 2)
    p.kappa = np.ones(p.U.shape, np.float32)
    p.rinv_v = np.ones(p.V.shape, np.float32)
    p.rinv_w = np.ones(p.W.shape, np.float32)
    b = run_gpu(adi, p, 2)
    assert_parity(b, a, tol=1e-14, what="constant media")


def test_media_mms_gpu(adi):
    """The medium MMS on the GPU: parity with the oracle at N = 256 (fp32 media) after
    90 steps, and the oracle's convergence rate continued to N = 512.  (Parity is
    checked mid-period: at t = T the exact velocities vanish, V and W are pure
    discretisation error, and a relative norm of them is ill-conditioned.)"""
    errs = []
    for N in (128, 256, 512):
        p = medium_mms_problem(MFD, N + 1, t_sim=MediumMMS().T, f32=True)
        s = adi.AdiSolver.from_problem(p)
        nst = p.meta["steps"]
        if N == 256:
            s.step(90)
            assert_parity(s.get_fields(), run_oracle(p, 90), what="medium MMS 256, 90 steps")
            s.step(nst - 90)
        else:
            s.step(nst)
        g = s.get_fields()
        s.close()
        errs.append(medium_error(p, g[0], p.meta["t_end"]))
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert all(r >= 0.9 for r in rates), (errs, rates)


def test_media_api_errors(adi):
    p = random_problem(MFD, 41, seed=1, steps=2, media=True)
    s = adi.AdiSolver.from_problem(p)
    with pytest.raises(adi.AdiError):
        s.set_media(p.kappa, None, p.rinv_w)
    bad = p.kappa.copy()
    bad[5, 5] = -1.0
    with pytest.raises(adi.AdiError):
        s.set_media(bad, p.rinv_v, p.rinv_w)
    s.set_param(adi.ADI_EPS, 1e-8)
    with pytest.raises(adi.AdiError):
        s.step(1)
    s.set_param(adi.ADI_EPS, 0.0)
    s.step(1)
    # back to the scalar medium (second step, t = dt)
    s.set_media(None, None, None)
    s.set_fields(p.U, p.V, p.W)
    s.step(1)
    g = s.get_fields()
    s.close()
    kw = p.oracle_kwargs()
    for k in ("kappa", "rinv_v", "rinv_w"):
        kw.pop(k)
    o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, m0=1, nsteps=1, **kw)
    assert_parity(g, o, what="media cleared")


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n,chunks", [(301, 16), (517, 6)])
def test_media_forced_segments(adi, method, n, chunks):
    """Forced multi-segment tilings (halos on a small grid) with media."""
    p = random_problem(method, n, seed=n + chunks, steps=2, media=True)
    s = adi.AdiSolver.from_problem(p)
    s.set_param(adi.ADI_TILE_CHUNKS, chunks)
    s.step(2)
    g = s.get_fields()
    s.close()
    assert_parity(g, run_oracle(p, 2), what=f"media {n} chunks={chunks}")
