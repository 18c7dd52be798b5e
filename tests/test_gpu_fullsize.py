"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py
times: element by element against the oracle, relative L2 <= 1e-12 and relative
max-norm <= 1e-11 per field (tests/parity.py).

* config 4: the single 16384^2-node grid of the Γ = 0 harmonic MMS (eq. 11,
  PAPER.md:399-407), K = 8, default tiling, both methods, 2 steps in one call (the
  prologue, an ADI-rows launch, an ADI-columns launch whose epilogue is the next
  step's stage-1 terms, and the FINAL columns launch: every kernel kind the bench
  times).  SURVEY §8d item 4 asks for one- and few-step parity at this size.
* config 5: shot 0 of a batch of 8 Ricker shots at 4096^2 nodes over 100 steps
  (SURVEY §8d item 5), in the batched handle bench.py --shots times.

The oracle needs ~40 GB of host memory at 16384^2; the test skips on a smaller host.
"""
import numpy as np
import pytest

import oracle
from adi_inputs import CFD, MFD, MMS, mms_problem, ricker_problem
from parity import check

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = 1e-12


@pytest.fixture(scope="module")
def adi():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2006_07583_b200 as m
    m.lib()
    return m


def host_gb():
    try:
        import psutil
        return psutil.virtual_memory().available / 2 ** 30
    except Exception:
        return 0.0


@pytest.mark.parametrize("method", [MFD, CFD])
def test_config4_parity_16384(adi, method):
    if host_gb() < 64:
        pytest.skip(f"needs ~64 GB of free host memory (have {host_gb():.0f} GB)")
    n, steps = 16384, 2
    p = mms_problem(method, n, MMS(), steps=steps + 1, K=8)
    s = adi.AdiSolver.from_problem(p)
    s.step(steps)
    g = s.get_fields()
    s.close()
    o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=steps,
                   **p.oracle_kwargs())
    for name, a, b in zip("UVW", g, o):
        assert np.isfinite(a).all()
        check(a, b, what=f"config4 {('CFD', 'MFD')[method]}", name=name)


def test_config5_shot0_parity_4096(adi):
    n, B, steps = 4096, 8, 100
    probs = [ricker_problem(n, shot=s, nshots=64, steps=steps) for s in range(B)]
    p0 = probs[0]
    s = adi.AdiSolver(n, n, p0.h, p0.dt, 1.0, MFD, batch=B)
    s.set_point_sources([p.src[0] for p in probs], [p.src[1] for p in probs], p0.gf)
    s.set_fields(np.zeros((B,) + p0.U.shape), np.zeros((B,) + p0.V.shape), np.zeros((B,) + p0.W.shape))
    s.step(steps)
    U, V, W = s.get_fields()
    s.close()
    o = oracle.run(p0.method, p0.nx, p0.ny, p0.h, p0.dt, p0.c, p0.K, p0.U, p0.V, p0.W, nsteps=steps,
                   **p0.oracle_kwargs())
    assert np.abs(o[0]).max() > 0
    for name, a, b in zip("UVW", (U[0], V[0], W[0]), o):
        check(a, b, what="config5 shot 0", name=name)
    # the other shots (no oracle run each): the step is translation invariant away from
    # the walls, so shot j is shot 0 moved by its source offset d = ix_j - ix_0 columns.
    # Checked in max-norm on a 701-column window around each source (100 steps at cfl
    # 0.81 travel 81 cells; the window stays >= 60 cells from the side walls, ~270 cells
    # beyond the wavefront, where the implicit sweeps' tails are far below round-off)
    ix0 = probs[0].src[0]
    c0, c1 = ix0 - 350, ix0 + 351
    assert c0 >= 60
    for j in range(1, B):
        d = probs[j].src[0] - ix0
        assert probs[j].src[1] == probs[0].src[1] and c1 + d <= n - 60
        assert np.isfinite(U[j]).all()
        for name, a, b in (("U", U[j][:, c0 + d:c1 + d], U[0][:, c0:c1]),
                           ("V", V[j][:, c0 + d:c1 + d], V[0][:, c0:c1]),
                           ("W", W[j][:, c0 + d:c1 + d], W[0][:, c0:c1])):
            check(a, b, what=f"config5 shot {j} = shot 0 shifted by {d}", name=name)
