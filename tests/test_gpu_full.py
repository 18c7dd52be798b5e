"""GPU parity of the full-matrix CFD variant with a Cerjan layer (SURVEY §8f row
f4, ADI_CFD_FULL) against oracle.run_full, through the C-ABI: relative L2 <= 1e-12
per field on seeded random states (every node), dense and point sources, with and
without the absorbing layer, over the generic tiles (short lines), the lean tiles
with line ends (1601^2), rectangles and split calls; plus the API's error paths."""
import numpy as np
import pytest

import oracle

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


def problem(nx, ny, steps, seed, cfl=0.91, source=True):
    rng = np.random.default_rng(seed)
    h = 1.0 / (max(nx, ny) - 1)
    U, V, W = (rng.standard_normal((ny, nx)) for _ in range(3))
    phi = rng.standard_normal((ny, nx)) if source else None
    gf = rng.standard_normal(2 * steps + 1)
    return dict(nx=nx, ny=ny, h=h, dt=cfl * h, U=U, V=V, W=W, phi=phi, gf=gf)


def run_gpu(adi, q, split, nb=0, a=0.015, src=None, K=8):
    s = adi.AdiSolver(q["nx"], q["ny"], q["h"], q["dt"], 1.0, adi.ADI_CFD_FULL, K=K)
    s.set_fields(q["U"], q["V"], q["W"])
    s.set_source(q["phi"], src, q["gf"])
    if nb:
        s.set_param(adi.ADI_ABSORB_WIDTH, nb)
        s.set_param(adi.ADI_ABSORB_RATE, a)
    for k in split:
        s.step(k)
    out = s.get_fields()
    s.close()
    return out


def run_oracle(q, steps, nb=0, a=0.015, src=None, K=8):
    return oracle.run_full(q["nx"], q["ny"], q["h"], q["dt"], 1.0, K, q["U"], q["V"], q["W"], phi=q["phi"],
                           gf=q["gf"], src=src, nsteps=steps, nb=nb, a=a)


@pytest.mark.parametrize("n,steps", [(21, 4), (41, 3), (333, 2)])
@pytest.mark.parametrize("nb", [0, 6])
def test_full_parity_generic_tiles(adi, n, steps, nb):
    q = problem(n, n, steps, seed=n + nb)
    assert_parity(run_gpu(adi, q, [steps], nb=nb, a=0.05), run_oracle(q, steps, nb=nb, a=0.05),
                  what=f"full {n} nb={nb}")


@pytest.mark.parametrize("nb", [0, 20])
def test_full_parity_lean_tiles(adi, nb):
    q = problem(1601, 1601, 3, seed=5 + nb)
    assert_parity(run_gpu(adi, q, [1, 2], nb=nb), run_oracle(q, 3, nb=nb), what=f"full 1601 nb={nb}")


@pytest.mark.parametrize("nx,ny", [(77, 2100), (2101, 1602)])
def test_full_parity_rectangles(adi, nx, ny):
    q = problem(nx, ny, 2, seed=nx)
    assert_parity(run_gpu(adi, q, [2], nb=20), run_oracle(q, 2, nb=20), what=f"full {nx}x{ny}")


def test_full_point_source_and_split_calls(adi):
    q = problem(1601, 1601, 4, seed=9, source=False)
    src = (0, 700)   # a boundary node: the full variant's pressure is unknown there too
    assert_parity(run_gpu(adi, q, [1, 1, 2], nb=20, src=src), run_oracle(q, 4, nb=20, src=src),
                  what="full point source")


def test_full_absorbs_on_gpu(adi):
    """The oracle's absorption pin, continued on the GPU at 1025^2: a centred pulse
    leaves less than 1 % of its energy after crossing a 40-point layer."""
    n, steps = 1025, 1800
    h = 1.0 / (n - 1)
    x = np.linspace(0, 1, n)
    X, Y = np.meshgrid(x, x)
    U0 = np.exp(-((X - 0.5) ** 2 + (Y - 0.5) ** 2) / (2 * 0.04 ** 2))
    Z = np.zeros((n, n))
    s = adi.AdiSolver(n, n, h, 0.5 * h, 1.0, adi.ADI_CFD_FULL)
    s.set_fields(U0, Z, Z)
    s.set_param(adi.ADI_ABSORB_WIDTH, 40)
    s.set_param(adi.ADI_ABSORB_RATE, 0.0075)
    s.step(steps)
    U, V, W = s.get_fields()
    s.close()
    e = np.sum(U ** 2 + V ** 2 + W ** 2) / np.sum(U0 ** 2)
    assert e < 0.01, e


def test_full_api_errors(adi):
    q = problem(41, 41, 2, seed=1)
    s = adi.AdiSolver(41, 41, q["h"], q["dt"], 1.0, adi.ADI_CFD_FULL)
    assert s.su == s.sv == s.sw == (41, 41)
    with pytest.raises(adi.AdiError):
        s.set_boundary((np.ones(41), np.ones(41), np.ones(41), np.ones(41)), None)
    with pytest.raises(adi.AdiError):
        s.set_param(adi.ADI_ABSORB_WIDTH, 21)    # > min(nx, ny) / 2
    with pytest.raises(adi.AdiError):
        adi.adi_set_band(s.handle, 0, 20)
    s.set_param(adi.ADI_EPS, 1e-8)
    s.set_fields(q["U"], q["V"], q["W"])
    with pytest.raises(adi.AdiError):
        s.step(1)
    s.close()
    r = adi.AdiSolver(41, 41, q["h"], q["dt"], 1.0, adi.ADI_CFD)
    with pytest.raises(adi.AdiError):
        r.set_param(adi.ADI_ABSORB_WIDTH, 5)     # the layer belongs to the full variant
    r.close()


def test_full_batch(adi):
    """A batch of 2 full-variant grids (shared source pattern and layer)."""
    n, B, steps = 1601, 2, 2
    qs = [problem(n, n, steps, seed=30 + b) for b in range(B)]
    q0 = qs[0]
    s = adi.AdiSolver(n, n, q0["h"], q0["dt"], 1.0, adi.ADI_CFD_FULL, batch=B)
    s.set_fields(np.stack([q["U"] for q in qs]), np.stack([q["V"] for q in qs]), np.stack([q["W"] for q in qs]))
    s.set_source(q0["phi"], None, q0["gf"])
    s.set_param(adi.ADI_ABSORB_WIDTH, 20)
    s.step(steps)
    g = s.get_fields()
    s.close()
    for b, q in enumerate(qs):
        o = oracle.run_full(n, n, q0["h"], q0["dt"], 1.0, 8, q["U"], q["V"], q["W"], phi=q0["phi"], gf=q0["gf"],
                            nsteps=steps, nb=20)
        assert_parity([x[b] for x in g], o, what=f"full batch member {b}")


@pytest.mark.parametrize("n,chunks,K", [(301, 16, 8), (517, 6, 3)])
def test_full_forced_segments(adi, n, chunks, K):
    """Forced multi-segment tilings (ADI_TILE_CHUNKS: 64-point halos on a small grid)
    and K != 8."""
    q = problem(n, n, 3, seed=n + chunks)
    s = adi.AdiSolver(n, n, q["h"], q["dt"], 1.0, adi.ADI_CFD_FULL, K=K)
    s.set_param(adi.ADI_TILE_CHUNKS, chunks)
    s.set_fields(q["U"], q["V"], q["W"])
    s.set_source(q["phi"], None, q["gf"])
    s.set_param(adi.ADI_ABSORB_WIDTH, 12)
    s.step(3)
    g = s.get_fields()
    s.close()
    assert_parity(g, run_oracle(q, 3, nb=12, K=K), what=f"full {n} chunks={chunks} K={K}")
