"""ADI_GRAPH (include/adi.h): adi_step(n) captured into one CUDA graph.  The same kernels
with the same parameters run, so the results are bitwise those of plain launches, and
the oracle's at the parity bar; one host launch per call (the short lines of configs 1-2
are launch-bound)."""
import numpy as np
import pytest

import oracle
from adi_inputs import CFD, MFD, random_problem, ricker_problem
from parity import assert_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def adi():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2006_07583_b200 as m
    m.lib()
    return m


def run(adi, p, split, graph, stream=None, **params):
    s = adi.AdiSolver.from_problem(p, stream=stream)
    s.set_param(adi.ADI_GRAPH, graph)
    for k, v in params.items():
        s.set_param(getattr(adi, k), v)
    h0 = s.stats()["host_launches"]
    for k in split:
        s.step(k)
    hl = s.stats()["host_launches"] - h0
    out = s.get_fields()
    s.close()
    return out, hl


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n", [41, 333, 1601])
def test_graph_bitwise_and_parity(adi, method, n):
    split = [3, 1, 4]
    p = random_problem(method, n, seed=n + method, steps=sum(split))
    a, hl_a = run(adi, p, split, 1)
    b, hl_b = run(adi, p, split, 0)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    assert hl_a == len(split) and hl_b > 2 * sum(split)
    o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=sum(split), **p.oracle_kwargs())
    assert_parity(a, o, what=f"graph n={n}")


def test_graph_user_stream_timing_and_checks(adi):
    """On a user stream, with ADI_TIMING (event nodes inside the graph) and
    ADI_CHECK_FINITE (checked after the graph launch); carry off."""
    import torch
    p = random_problem(CFD, 1601, seed=3, steps=6)
    st = torch.cuda.Stream()
    a, _ = run(adi, p, [2, 4], 1, stream=st.cuda_stream, ADI_TIMING=1, ADI_CHECK_FINITE=1, ADI_CARRY=0)
    b, _ = run(adi, p, [2, 4], 0, ADI_CARRY=0)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    s = adi.AdiSolver.from_problem(p, stream=st.cuda_stream)
    s.set_param(adi.ADI_GRAPH, 1)
    s.set_param(adi.ADI_TIMING, 1)
    s.step(3)
    kt = s.kernel_times()
    s.close()
    assert kt["row"][1] == 3 and kt["row"][0] > 0


def test_graph_batch_point_sources_media(adi):
    n, B, steps = 1601, 2, 4
    probs = [ricker_problem(n, shot=s, nshots=4, steps=steps, f0=20.0, t0=0.05) for s in range(B)]
    p0 = probs[0]
    rng = np.random.default_rng(1)
    med = [rng.uniform(0.6, 1.0, x.shape).astype(np.float32) for x in (p0.U, p0.V, p0.W)]
    outs = []
    for graph in (1, 0):
        s = adi.AdiSolver(n, n, p0.h, p0.dt, 1.0, MFD, batch=B)
        s.set_param(adi.ADI_GRAPH, graph)
        s.set_fields(np.stack([p.U for p in probs]) + 1.0, np.stack([p.V for p in probs]),
                     np.stack([p.W for p in probs]))
        s.set_point_sources([p.src[0] for p in probs], [p.src[1] for p in probs], p0.gf)
        s.set_media(*med)
        s.step(2)
        s.step(2)
        outs.append(s.get_fields())
        s.close()
    for x, y in zip(*outs):
        assert np.array_equal(x, y)


def test_graph_split_calls_carry(adi):
    """Carry across graph calls (the captured last column kernel writes the next a2)."""
    p = random_problem(MFD, 1601, seed=9, steps=3)
    a, _ = run(adi, p, [3], 1)
    b, _ = run(adi, p, [3], 0)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
