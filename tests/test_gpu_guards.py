"""Out-of-bounds writes, checked without compute-sanitizer (which this pool does not run):
with ADI_GUARD_CHECK=1 every field array's guard regions hold a canary pattern, and
adi_check_guards counts overwritten guard words.  Every kernel kind runs here -- lean and
generic tiles, the carry kernel, FINAL, the warp- and thread-per-line kernels, media, the full-matrix
variant, the stopping rule, graph capture, the async stores, band-local re-layouts and both
dist-local decompositions -- and no guard word may change.  The results must also equal
those of zero guards bit for bit (no result depends on what lies beyond an array)."""
import os

import numpy as np
import pytest

from adi_inputs import CFD, MFD, random_problem

pytestmark = pytest.mark.gpu


@pytest.fixture()
def adi():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2006_07583_b200 as m
    m.lib()
    os.environ["ADI_GUARD_CHECK"] = "1"
    yield m
    os.environ.pop("ADI_GUARD_CHECK", None)


def _plain(adi, p, params, plan):
    s = adi.AdiSolver.from_problem(p)
    for k, v in params:
        s.set_param(getattr(adi, k), v)
    for a in plan:
        s.step(a) if isinstance(a, int) else s.set_param(getattr(adi, a[0]), a[1])
    out = s.get_fields()
    bad = adi.adi_check_guards(s.handle)
    s.close()
    return out, bad


CASES = [("lean", 1601, [], [2, 1, ("ADI_CARRY", 0), 1]),
         ("generic", 333, [("ADI_THREAD_LINES", 0)], [2, 1]),
         ("warp", 41, [("ADI_THREAD_LINES", 1)], [2, 1]),
         ("warp12", 321, [("ADI_THREAD_LINES", 1)], [2, 1]),
         ("thread", 41, [("ADI_THREAD_LINES", 1), ("ADI_WARP_LINES", 0)], [2, 1]),
         ("segments", 1001, [("ADI_TILE_CHUNKS", 12)], [2]),
         ("frag", 2101, [], [2, 1]),   # MFD: the fragment plan (4 lines per warp)
         ("graph", 1601, [("ADI_GRAPH", 1)], [2, 2]),
         ("async", 2101, [("ADI_ASYNC_STORE", 1)], [2, 1]),
         ("stop", 333, [("ADI_K_SWEEPS", 10), ("ADI_EPS", 1e-6), ("ADI_K_MIN", 3)], [2])]


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("case", [c[0] for c in CASES])
def test_no_guard_word_written(adi, method, case):
    _, n, params, plan = next(c for c in CASES if c[0] == case)
    p = random_problem(method, n, seed=n, steps=8, media=(case == "generic"))
    out, bad = _plain(adi, p, params, plan)
    assert bad == 0, (case, bad)
    os.environ.pop("ADI_GUARD_CHECK")
    ref, _ = _plain(adi, p, params, plan)
    os.environ["ADI_GUARD_CHECK"] = "1"
    for a, b in zip(out, ref):
        assert np.array_equal(a, b)


def test_no_guard_word_written_full_bands_dist(adi):
    n = 1601
    rng = np.random.default_rng(0)
    h = 1.0 / (n - 1)
    s = adi.AdiSolver(n, n, h, 0.91 * h, 1.0, adi.ADI_CFD_FULL)
    s.set_fields(*(rng.standard_normal((n, n)) for _ in range(3)))
    s.set_source(rng.standard_normal((n, n)), None, rng.standard_normal(9))
    s.set_param(adi.ADI_ABSORB_WIDTH, 20)
    s.step(2)
    assert adi.adi_check_guards(s.handle) == 0
    s.close()
    for method in (CFD, MFD):
        p = random_problem(method, 2101, seed=3, steps=4)
        s = adi.AdiSolver.from_problem(p)
        y0, y1, halo, npos = adi.adi_band_info(s.handle)
        adi.adi_set_band(s.handle, npos // 3, 2 * npos // 3)   # re-layout to band-local arrays
        s.step(1)
        assert adi.adi_check_guards(s.handle) == 0
        s.close()
        for mode, fused in ((adi.ADI_DIST_HALO, 0), (adi.ADI_DIST_TRANSPOSE, 1), (adi.ADI_DIST_TRANSPOSE, 0)):
            hs = adi.adi_create_dist_local(p.nx, p.ny, p.h, p.dt, p.c, method, 1, 3, mode)
            ss = [adi.AdiSolver.adopt(x, p.nx, p.ny, p.h, p.dt, p.c, method) for x in hs]
            for x in ss:
                if mode == adi.ADI_DIST_TRANSPOSE:
                    x.set_param(adi.ADI_DIST_FUSED, fused)   # the peer stores / the all-to-all
                x.set_fields(p.U, p.V, p.W)
                x.set_source(p.phi, None, p.gf)
                x.set_boundary(p.edges, p.gb)
            adi.adi_step_dist_local(hs, 2)
            adi.adi_step_dist_local(hs, 1)
            for x in ss:
                assert adi.adi_check_guards(x.handle) == 0, mode
                x.close()
