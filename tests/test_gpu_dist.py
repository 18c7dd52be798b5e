"""Band decomposition (multi-GPU design) verified on one GPU:
P ranks emulated in one process (LocalGroup: ranks run one after another,
halo messages are device copies).  The gathered result must equal the
single-handle result and the oracle to 1e-12."""
import numpy as np
import pytest

import oracle
from adi_inputs import CFD, MFD, random_problem, ricker_problem

from parity import check, rel  # noqa: E402,F401  (rel L2 + rel max)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def adi():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2006_07583_b200 as m
    m.lib()
    return m


def make_group(adi, p, world, **kw):
    from paper_2006_07583_b200 import dist
    solvers = [adi.AdiSolver.from_problem(p, **kw) for _ in range(world)]
    y0, y1, halo, npos = adi.adi_band_info(solvers[0].handle)
    bands = dist.band_partition(npos, world, halo)
    return dist.LocalGroup(solvers, bands), solvers


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n,world,split", [(301, 2, [3]), (517, 3, [2, 2]), (1601, 4, [1, 1]),
                                            (2101, 8, [2])])
def test_band_group_equals_single_and_oracle(adi, method, n, world, split):
    steps = sum(split)
    p = random_problem(method, n, seed=n + world, steps=steps)
    g, solvers = make_group(adi, p, world)
    for k in split:          # several calls: exercises the U/W halo exchange too
        g.step(k)
    got = g.gather()
    s = adi.AdiSolver.from_problem(p)
    s.step(steps)
    ref = s.get_fields()
    o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=steps,
                   **p.oracle_kwargs())
    for name, a, b, c in zip("UVW", got, ref, o):
        check(a, b)
        check(a, c)


def test_band_group_batch_shots(adi):
    """Config-5 style batch of shots inside a band-decomposed grid."""
    from paper_2006_07583_b200 import dist
    n, B, steps = 257, 3, 12
    probs = [ricker_problem(n, shot=s, nshots=B, steps=steps, f0=12.0, t0=0.1) for s in range(B)]
    p0 = probs[0]

    def mk():
        s = adi.AdiSolver(n, n, p0.h, p0.dt, 1.0, MFD, batch=B)
        s.set_fields(np.stack([p.U for p in probs]), np.stack([p.V for p in probs]),
                     np.stack([p.W for p in probs]))
        s.set_point_sources([p.src[0] for p in probs], [p.src[1] for p in probs], p0.gf)
        return s
    solvers = [mk() for _ in range(2)]
    y0, y1, halo, npos = adi.adi_band_info(solvers[0].handle)
    g = dist.LocalGroup(solvers, dist.band_partition(npos, 2, halo))
    g.step(steps)
    got = g.gather()
    for b, p in enumerate(probs):
        o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=steps,
                       **p.oracle_kwargs())
        for a, c in zip(got, o):
            check(a[b], c)


@pytest.mark.parametrize("method", [CFD, MFD])
def test_band_group_with_media(adi, method):
    """Heterogeneous media (f3) inside the band decomposition: each band's handle holds
    the whole medium; the gathered result equals the oracle."""
    n, world, split = 1601, 3, [1, 1]
    p = random_problem(method, n, seed=77, steps=sum(split), media=True)
    g, solvers = make_group(adi, p, world)
    for k in split:
        g.step(k)
    got = g.gather()
    o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=sum(split),
                   **p.oracle_kwargs())
    for name, a, c in zip("UVW", got, o):
        check(a, c)


@pytest.mark.parametrize("method", [CFD, MFD])
def test_create_dist_single_rank(adi, method):
    """adi_create_dist with nranks = 1 is a plain handle: parity with the oracle through
    the same set/step/get calls (the multi-rank NCCL exchange needs one GPU per rank)."""
    p = random_problem(method, 1601, seed=21, steps=2)
    hd, rc = adi.adi_create_dist(p.nx, p.ny, p.h, p.dt, p.c, method, 1, None, 0, 1)
    assert rc >= 0
    adi.adi_set_fields(hd, p.U, p.V, p.W)
    adi.adi_set_source(hd, p.phi, -1, -1, p.gf)
    adi.adi_set_boundary(hd, p.edges, p.gb)
    adi.adi_step(hd, 2)
    import numpy as np
    from adi_inputs import shapes
    out = [np.zeros(s) for s in shapes(method, p.nx, p.ny)]
    adi.adi_get_fields(hd, *out)
    adi.adi_destroy(hd)
    o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=2, **p.oracle_kwargs())
    for name, a, c in zip("UVW", out, o):
        check(a, c)
