"""GPU parity of the inner stopping rule (Alg. 3/4, PAPER.md:652-721,
388-393): for the same eps the GPU picks the same sweep count per stage as the oracle
and the fields agree at 1e-12.  eps is placed between two consecutive test values of the
first row stage (no near-ties)."""
import numpy as np
import pytest

import oracle
from adi_inputs import CFD, MFD, random_problem

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


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n", [77, 1601])
def test_stopping_rule_matches_oracle(adi, method, n):
    steps, K, kmin = 3, 12, 3
    p = random_problem(method, n, seed=21, steps=steps)
    p.K = K
    kw = p.oracle_kwargs()
    info = {}
    oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, K, p.U, p.V, p.W, nsteps=1, eps=1e300, kmin=kmin,
               info=info, **kw)
    t = info["tests"][0, 0]
    mid = (kmin + K) // 2
    eps = float(np.sqrt(t[mid] * t[mid + 1]))
    info = {}
    o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, K, p.U, p.V, p.W, nsteps=steps, eps=eps,
                   kmin=kmin, info=info, **kw)
    s = adi.AdiSolver.from_problem(p)
    s.set_param(adi.ADI_EPS, eps)
    s.set_param(adi.ADI_K_MIN, kmin)
    for st in range(steps):
        s.step(1)
        assert adi.adi_get_last_sweeps(s.handle) == tuple(int(k) for k in info["k"][st]), st
        # adi_get_stats: the last-sweep residuals (the Alg. 3/4 test at the chosen k)
        stt = s.stats()
        for stage in range(2):
            k = int(info["k"][st, stage])
            assert stt["last_k"][stage] == k
            assert stt["last_test"][stage] == pytest.approx(info["tests"][st, stage, k], rel=1e-10)
    g = s.get_fields()
    s.close()
    assert kmin < info["k"][0, 0] < K           # the rule actually stopped early
    for name, a, b in zip("UVW", g, o):
        check(a, b, name=name)


def test_eps_zero_reports_fixed_sweeps(adi):
    p = random_problem(MFD, 41, seed=2, steps=1)
    s = adi.AdiSolver.from_problem(p)
    s.step(1)
    assert adi.adi_get_last_sweeps(s.handle) == (p.K, p.K)
    stt = s.stats()
    assert stt["last_test"] == [-1.0, -1.0] and stt["last_k"] == [p.K, p.K]
    s.close()


def test_stopping_rule_rejects_bands(adi):
    p = random_problem(MFD, 301, seed=2, steps=1)
    s = adi.AdiSolver.from_problem(p)
    s.set_param(adi.ADI_EPS, 1e-3)
    adi.adi_set_band(s.handle, 0, 150)
    with pytest.raises(adi.AdiError):
        s.step(1)
    s.close()
