"""GPU parity: the CUDA path (through the C-ABI) against the oracle, element by
element on the same seeded inputs.  Tolerance: relative L2 <= 1e-12 per field
(BASELINE.json north_star) and relative max-norm <= 1e-11 (tests/parity.py).  CFD runs are limited to horizons where round-off
amplification of the literal CFD reading stays below that bound (DESIGN.md §4,
SURVEY §8c P10); the 200-step config-1 run is checked against the oracle's own
round-off sensitivity instead."""
import math

import numpy as np
import pytest

import oracle
from adi_inputs import CFD, MFD, MMS, mms_problem, random_problem, ricker_problem
from parity import assert_parity, check, rel  # noqa: F401  (rel L2 + rel max)

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


def run_oracle(p, nsteps, **over):
    kw = p.oracle_kwargs()
    kw.update(over)
    return oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=nsteps, **kw)


def run_gpu(adi, p, nsteps, chunks=0, split=None, thread=-1):
    s = adi.AdiSolver.from_problem(p)
    s.set_param(adi.ADI_THREAD_LINES, thread)
    if chunks:
        s.set_param(adi.ADI_TILE_CHUNKS, chunks)
    if split:
        for k in split:
            s.step(k)
    else:
        s.step(nsteps)
    out = s.get_fields()
    s.close()
    return out


def oracle_sensitivity(p, nsteps, o):
    """Relative change of the oracle's result when U0 is perturbed by 1 ulp."""
    import copy
    q = copy.copy(p)
    q.U = p.U * (1 + 2.0 ** -52)
    o2 = run_oracle(q, nsteps)
    return [rel(c, b) for c, b in zip(o2, o)]


@pytest.mark.parametrize("thread", [0, 1])
@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n", [9, 17, 33, 41, 100])
def test_random_parity_small(adi, method, n, thread):
    """Random state, dense source, boundary data; single-tile lines incl. N=8 and ragged ends;
    the warp-per-line generic tiles (thread 0) and the thread-per-line kernels (1)."""
    p = random_problem(method, n, seed=n, steps=3)
    assert_parity(run_gpu(adi, p, 3, thread=thread), run_oracle(p, 3), what=f"n={n} thread={thread}")


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n,ny", [(41, 41), (77, 130), (257, 257), (130, 9)])
def test_thread_kernels_rectangles_batch_points(adi, method, n, ny):
    """Thread-per-line kernels: rectangles, the largest forced size, split
    calls (each call's prologue), a batch with point sources; rel L2 and max-norm."""
    p = random_problem(method, n, seed=n + ny, steps=5, ny=ny)
    assert_parity(run_gpu(adi, p, 5, split=[2, 3], thread=1), run_oracle(p, 5), what=f"thread {n}x{ny}")
    B = 2
    probs = [random_problem(method, n, seed=40 + b, steps=3, ny=ny) for b in range(B)]
    s = adi.AdiSolver(n, ny, probs[0].h, probs[0].dt, 1.0, method, batch=B)
    s.set_param(adi.ADI_THREAD_LINES, 1)
    s.set_fields(np.stack([q.U for q in probs]), np.stack([q.V for q in probs]), np.stack([q.W for q in probs]))
    ix, iy = [3, n // 2], [ny // 3, 2]
    s.set_point_sources(ix, iy, probs[0].gf)
    s.step(3)
    got = s.get_fields()
    s.close()
    for b, q in enumerate(probs):
        o = oracle.run(q.method, q.nx, q.ny, q.h, q.dt, q.c, q.K, q.U, q.V, q.W, nsteps=3,
                       src=(ix[b], iy[b]), gf=probs[0].gf)
        assert_parity([x[b] for x in got], o, what=f"thread batch {b}")


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n,chunks", [(301, 16), (517, 17), (1001, 20)])
def test_random_parity_segmented(adi, method, n, chunks):
    """Forced multi-segment tiling with halos: still exact to round-off."""
    p = random_problem(method, n, seed=3 * n, steps=2)
    assert_parity(run_gpu(adi, p, 2, chunks=chunks), run_oracle(p, 2), what=f"n={n} cap={chunks}")


@pytest.mark.parametrize("method", [CFD, MFD])
def test_parity_default_tiling_large(adi, method):
    """A grid whose column sweep is segmented by the default planner (lines > 1024 points)."""
    p = random_problem(method, 1601, seed=5, steps=1)
    assert_parity(run_gpu(adi, p, 1), run_oracle(p, 1), what="1601")


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n", [1601, 1602, 2100, 2101])
def test_parity_lean_line_ends(adi, method, n):
    """Lean tiles at the line ends: the first segment starts at the
    line start, the last ends at position n (even n+1 - 1024) or n+1 (odd); closures
    (MFD) and the rank <= 3 end corrections of the constant-pivot solve (CFD)."""
    p = random_problem(method, n, seed=7 * n, steps=2)
    assert_parity(run_gpu(adi, p, 2), run_oracle(p, 2), what=f"n={n}")


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("K", [1, 2, 8, 13])
def test_parity_sweeps(adi, method, K):
    p = random_problem(method, 29, seed=K, steps=2)
    p.K = K
    assert_parity(run_gpu(adi, p, 2), run_oracle(p, 2), what=f"K={K}")


@pytest.mark.parametrize("method", [CFD, MFD])
def test_split_calls_equal_one_call(adi, method):
    """adi_step(2)+adi_step(3) equals adi_step(5) (state is canonical between calls)."""
    p = random_problem(method, 37, seed=2, steps=5)
    a = run_gpu(adi, p, 5)
    b = run_gpu(adi, p, 5, split=[2, 3])
    assert_parity(b, a, tol=1e-13)
    assert_parity(a, run_oracle(p, 5))


@pytest.mark.parametrize("thread", [0, 1])
def test_mfd_mms_ladder_parity(adi, thread):
    """Config 2: MFD, Γ=0, 5T, cfl 0.81, K=8 on 41, 81, 161 nodes — full runs, with the
    tile kernels and with the thread-per-line kernels.
    At t = 5T the exact V̄, W̄ vanish (∝ sin ωt), so their relative error is
    judged against the oracle's own sensitivity; U at 1e-12 outright."""
    T = 1 / math.sqrt(2)
    for n in (41, 81, 161):
        p = mms_problem(MFD, n, MMS(), t_sim=5 * T)
        st = p.meta["steps"]
        g, o = run_gpu(adi, p, st, thread=thread), run_oracle(p, st)
        assert rel(g[0], o[0]) <= TOL
        assert_parity(g, o, what=f"MFD MMS n={n}", floor=oracle_sensitivity(p, st, o))


@pytest.mark.parametrize("n,steps", [(41, 100), (81, 200), (161, 350)])
def test_mfd_mms_midrun_parity(adi, n, steps):
    """Config 2 at a mid-run time where every field is O(10): strict 1e-12."""
    p = mms_problem(MFD, n, MMS(), t_sim=5 / math.sqrt(2))
    assert_parity(run_gpu(adi, p, steps), run_oracle(p, steps), what=f"MFD MMS n={n} @{steps}")


@pytest.mark.parametrize("thread", [0, -1])
def test_cfd_config1_short_parity(adi, thread):
    """Config 1 (CFD 41x41, Γ=0, Δt = 0.91 h) for the first 60 steps at 1e-12
    (beyond ~75 steps the literal CFD reading has amplified round-off past 1e-12
    in ANY implementation: SURVEY fact 5-6)."""
    p = mms_problem(CFD, 41, MMS(), steps=200)
    assert_parity(run_gpu(adi, p, 60, thread=thread), run_oracle(p, 60), what="CFD config1 60 steps")


@pytest.mark.parametrize("thread", [0, -1])
def test_cfd_config1_full_within_roundoff_amplification(adi, thread):
    """Config 1 over all 200 steps, judged against the oracle's own 1-ulp
    sensitivity (x10 margin)."""
    p = mms_problem(CFD, 41, MMS(), steps=200)
    g, o = run_gpu(adi, p, 200, thread=thread), run_oracle(p, 200)
    assert_parity(g, o, what="CFD config1 200 steps", floor=oracle_sensitivity(p, 200, o))


def test_ricker_batch_parity(adi):
    """Config 5 shape: a batch of point-source shots, zero IC, free surface."""
    n, B, steps = 129, 4, 30
    probs = [ricker_problem(n, shot=s, nshots=B, steps=steps, f0=12.0, t0=0.1) for s in range(B)]
    p0 = probs[0]
    s = adi.AdiSolver(n, n, p0.h, p0.dt, 1.0, MFD, batch=B)
    s.set_fields(np.stack([p.U for p in probs]), np.stack([p.V for p in probs]),
                 np.stack([p.W for p in probs]))
    s.set_point_sources([p.src[0] for p in probs], [p.src[1] for p in probs], p0.gf)
    s.step(steps)
    U, V, W = s.get_fields()
    s.close()
    for b, p in enumerate(probs):
        o = run_oracle(p, steps)
        assert np.abs(o[0]).max() > 0
        assert_parity((U[b], V[b], W[b]), o, what=f"shot {b}")


@pytest.mark.parametrize("method", [CFD, MFD])
def test_zero_in_zero_out(adi, method):
    p = random_problem(method, 33, seed=0, steps=2, source=False, boundary=False)
    p.U[:] = 0
    p.V[:] = 0
    p.W[:] = 0
    U, V, W = run_gpu(adi, p, 2)
    assert not U.any() and not V.any() and not W.any()


def test_nonfinite_detected(adi):
    p = random_problem(MFD, 33, seed=0, cfl=1.3, steps=400, source=False, boundary=False)
    s = adi.AdiSolver.from_problem(p, check_finite=True)
    assert s.create_status == adi.ADI_WUNSTABLE
    with pytest.raises(adi.AdiError) as e:
        s.step(400)
    assert e.value.code == adi.ADI_ENONFINITE
    s.close()


def test_device_arrays_roundtrip(adi):
    import torch
    p = random_problem(MFD, 45, seed=9, steps=2)
    s = adi.AdiSolver.from_problem(p)
    dU, dV, dW = (torch.tensor(a, device="cuda") for a in (p.U, p.V, p.W))
    s.set_fields(dU, dV, dW)
    s.step(2)
    oU, oV, oW = (torch.empty_like(a) for a in (dU, dV, dW))
    s.get_fields_device(oU, oV, oW)
    torch.cuda.synchronize()
    assert_parity(tuple(a.cpu().numpy() for a in (oU, oV, oW)), run_oracle(p, 2))
    s.close()


@pytest.mark.parametrize("method", [CFD, MFD])
def test_async_transfers_equal_sync(adi, method):
    """adi_set_fields_async / adi_get_fields_async (pinned buffers, handle's own stream)
    give the same state as the synchronous calls."""
    import torch
    p = random_problem(method, 77, seed=11, steps=3)
    ref = run_gpu(adi, p, 3)
    st = torch.cuda.Stream()
    s = adi.AdiSolver.from_problem(p, stream=st.cuda_stream)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    hU, hV, hW = pin(p.U), pin(p.V), pin(p.W)
    oU, oV, oW = (torch.empty(x.shape, dtype=torch.float64).pin_memory().numpy() for x in (hU, hV, hW))
    adi.adi_set_fields_async(s.handle, hU, hV, hW)
    s.step(3)
    adi.adi_get_fields_async(s.handle, oU, oV, oW)
    st.synchronize()
    s.close()
    for name, a, b in zip("UVW", (oU, oV, oW), ref):
        assert np.array_equal(a, b), (name, rel(a, b), np.argwhere(a != b)[:5])


@pytest.mark.parametrize("method", [CFD, MFD])
def test_nonblocking_stream_equals_default(adi, method):
    """A handle on a non-blocking stream (torch streams are) gives bit-identical results:
    every set-up copy is ordered on the handle's stream and waited for (a plain
    cudaMemcpy from pageable memory may return before its DMA lands)."""
    import torch
    p = random_problem(method, 77, seed=11, steps=2)
    ref = run_gpu(adi, p, 2)
    for _ in range(6):
        st = torch.cuda.Stream()
        s = adi.AdiSolver.from_problem(p, stream=st.cuda_stream)
        s.step(2)
        got = s.get_fields()
        s.close()
        for name, a, b in zip("UVW", got, ref):
            assert np.array_equal(a, b), name


@pytest.mark.slow
@pytest.mark.parametrize("method,steps", [(CFD, 50), (MFD, 100)])
@pytest.mark.parametrize("k", [2, 9])
def test_config3_parity(adi, method, steps, k):
    """Γ = k ∈ {2, 9} (polynomial part of S, boundary S|∂Ω cos ωt,
    dense source with the polynomial part), 1601² nodes, parity after 50 (CFD) / 100 (MFD)
    steps against the oracle."""
    p = mms_problem(method, 1601, MMS(gamma=float(k), k=k), steps=steps)
    assert_parity(run_gpu(adi, p, steps), run_oracle(p, steps), what=f"config3 k={k}")


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("nx,ny", [(1601, 300), (77, 2100), (2101, 1602)])
def test_parity_rectangular_grids(adi, method, nx, ny):
    """nx != ny: the two sweep directions plan different tilings (lean and generic tiles)."""
    p = random_problem(method, nx, ny=ny, seed=nx + ny, steps=2)
    assert_parity(run_gpu(adi, p, 2), run_oracle(p, 2), what=f"{nx}x{ny}")


@pytest.mark.parametrize("method", [CFD, MFD])
def test_parity_batch_lean_tiles(adi, method):
    """A batch of 3 grids (shared source and boundary data) at 1601^2 (lean tiles)."""
    n, B, steps = 1601, 3, 2
    ps = [random_problem(method, n, seed=40 + b, steps=steps) for b in range(B)]
    p0 = ps[0]
    s = adi.AdiSolver(p0.nx, p0.ny, p0.h, p0.dt, p0.c, method, batch=B, K=p0.K)
    s.set_fields(np.stack([p.U for p in ps]), np.stack([p.V for p in ps]), np.stack([p.W for p in ps]))
    s.set_source(p0.phi, None, p0.gf)
    s.set_boundary(p0.edges, p0.gb)
    s.step(steps)
    g = s.get_fields()
    s.close()
    for b, p in enumerate(ps):
        o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=steps,
                       rho=p.rho, phi=p0.phi, gf=p0.gf, edges=p0.edges, gb=p0.gb)
        assert_parity([x[b] for x in g], o, what=f"batch member {b}")


@pytest.mark.parametrize("method", [CFD, MFD])
def test_parity_point_source_lean_tiles(adi, method):
    """Ricker point source on a 1601^2 grid (the source sits in a lean tile)."""
    p = ricker_problem(1601, shot=5, nshots=8, method=method, steps=6, f0=20.0, t0=0.05)
    assert_parity(run_gpu(adi, p, 6), run_oracle(p, 6), what="ricker 1601")


def test_parity_point_sources_batch_lean_tiles(adi):
    """A batch of shots with per-grid point sources (adi_set_point_sources) at 1601^2."""
    n, B, steps = 1601, 3, 4
    probs = [ricker_problem(n, shot=s, nshots=B, steps=steps, f0=20.0, t0=0.05) for s in range(B)]
    p0 = probs[0]
    s = adi.AdiSolver(n, n, p0.h, p0.dt, 1.0, MFD, batch=B)
    s.set_fields(np.stack([p.U for p in probs]), np.stack([p.V for p in probs]),
                 np.stack([p.W for p in probs]))
    s.set_point_sources([p.src[0] for p in probs], [p.src[1] for p in probs], p0.gf)
    s.step(steps)
    got = s.get_fields()
    s.close()
    for b, p in enumerate(probs):
        o = run_oracle(p, steps)
        assert_parity([x[b] for x in got], o, what=f"shot {b}")


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n,chunks,steps", [(1001, 12, 3), (2101, 16, 2)])
def test_segment_halo_is_exact(adi, method, n, chunks, steps):
    """The segment halo is exact to round-off: forced short segments
    (ADI_TILE_CHUNKS, many segment edges) against whole-line tiles on the GPU, max-norm
    relative difference <= 1e-14 per field (a halo deficit shows up far above that)."""
    p = random_problem(method, n, seed=n + chunks, steps=steps)
    a = run_gpu(adi, p, steps)
    b = run_gpu(adi, p, steps, chunks=chunks)
    for name, x, y in zip("UVW", a, b):
        d = np.abs(x - y).max() / np.abs(x).max()
        assert d <= 1e-14, (name, d)


@pytest.mark.parametrize("media", [False, True])
@pytest.mark.parametrize("method", [CFD, MFD])
def test_prefetch_knob_does_not_change_results(adi, method, media):
    """ADI_PREFETCH (an L2 prefetch distance, include/adi.h) is a performance knob:
    results are bitwise identical for every value; out-of-range values are refused."""
    outs = []
    p = random_problem(method, 2101, seed=4, steps=2, media=media)
    for v in (0, 1, 3):
        s = adi.AdiSolver.from_problem(p)
        s.set_param(adi.ADI_PREFETCH, v)
        s.step(2)
        outs.append(s.get_fields())
        s.close()
    for o in outs[1:]:
        for a, b in zip(o, outs[0]):
            assert np.array_equal(a, b)
    s = adi.AdiSolver.from_problem(p)
    for bad in (-1, 9, 1.5):
        with pytest.raises(adi.AdiError):
            s.set_param(adi.ADI_PREFETCH, bad)
    s.close()


def test_prefetch_knob_batch(adi):
    """ADI_PREFETCH with a batch (the prefetch target's grid z = batch index)."""
    n, B = 1601, 3
    probs = [random_problem(MFD, n, seed=30 + b, steps=2) for b in range(B)]
    p0 = probs[0]
    outs = []
    for v in (0, 2):
        s = adi.AdiSolver(n, n, p0.h, p0.dt, p0.c, MFD, batch=B)
        s.set_fields(np.stack([p.U for p in probs]), np.stack([p.V for p in probs]),
                     np.stack([p.W for p in probs]))
        s.set_source(p0.phi, None, p0.gf)
        s.set_boundary(p0.edges, p0.gb)
        s.set_param(adi.ADI_PREFETCH, v)
        s.step(2)
        outs.append(s.get_fields())
        s.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)


def _run_calls(adi, p, plan, carry, n_steps_table=None):
    """Run `plan` on one handle: ints are adi_step(n) calls, tuples are actions
    between calls ("get",), ("get_async",), ("source", phi, gf), ("fields", U, V, W),
    ("rho", v), ("boundary", edges, gb), ("points", ix, iy, gf), ("media", k, rv, rw),
    ("band", y0, y1)."""
    s = adi.AdiSolver.from_problem(p)
    s.set_param(adi.ADI_CARRY, carry)
    for a in plan:
        if isinstance(a, int):
            s.step(a)
        elif a[0] == "get":
            s.get_fields()
        elif a[0] == "get_async":
            import torch
            hs = [torch.empty(x.shape, dtype=torch.float64).pin_memory().numpy() for x in (p.U, p.V, p.W)]
            adi.adi_get_fields_async(s.handle, *hs)
            torch.cuda.synchronize()
        elif a[0] == "source":
            s.set_source(a[1], None, a[2])
        elif a[0] == "fields":
            s.set_fields(a[1], a[2], a[3])
        elif a[0] == "rho":
            s.set_param(adi.ADI_RHO, a[1])
        elif a[0] == "boundary":
            s.set_boundary(a[1], a[2])
        elif a[0] == "points":
            s.set_point_sources([a[1]], [a[2]], a[3])
        elif a[0] == "media":
            s.set_media(a[1], a[2], a[3])
        elif a[0] == "band":   # back to the whole grid (all y positions)
            adi.adi_set_band(s.handle, 0, adi.adi_band_info(s.handle)[3])
    out = s.get_fields()
    s.close()
    return out


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n", [37, 1601, 2101])
def test_carry_matches_one_call(adi, method, n):
    """ADI_CARRY (include/adi.h): the next call starts from the a2 computed by the previous
    call's last column kernel -- the one-call computation, so split calls match one call
    to rounding, with and without a get_fields in between; and the oracle at 1e-12."""
    p = random_problem(method, n, seed=7, steps=6)
    one = _run_calls(adi, p, [6], 1)
    split = _run_calls(adi, p, [2, ("get",), 1, 3], 1)
    nocarry = _run_calls(adi, p, [2, ("get",), 1, 3], 0)
    assert_parity(split, one, tol=1e-13)
    assert_parity(nocarry, one, tol=1e-13)
    assert_parity(split, run_oracle(p, 6))


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n", [1601, 2101])
def test_carry_invalidated_by_setters(adi, method, n):
    """A set_* call between two calls discards the carried a2: the result equals the
    same sequence with ADI_CARRY = 0 (a stale a2 would differ at O(dt)), in relative L2
    and in max-norm (line ends and segment seams included).  n = 2101: the line-end
    segments hold partial chunks.  A get_fields / get_fields_async between calls keeps
    the carry valid (same one-call result)."""
    p = random_problem(method, n, seed=8, steps=6)
    rng = np.random.default_rng(3)
    phi2 = rng.standard_normal(p.phi.shape)
    gf2 = rng.standard_normal(p.gf.shape)
    gb2 = rng.standard_normal(p.gb.shape)
    edges2 = tuple(rng.standard_normal(e.shape) for e in p.edges)
    U2, V2, W2 = (rng.standard_normal(a.shape) for a in (p.U, p.V, p.W))
    med = [rng.uniform(0.6, 1.0, a.shape).astype(np.float32) for a in (p.U, p.V, p.W)]
    ix, iy = p.U.shape[1] // 3, p.U.shape[0] // 2
    cases = ([("source", phi2, gf2)], [("fields", U2, V2, W2)], [("rho", 1.3)],
             [("boundary", edges2, gb2)], [("points", ix, iy, gf2)], [("media",) + tuple(med)],
             [("band",)], [("get",)], [("get_async",)])
    for between in cases:
        plan = [2] + between + [2]
        a = _run_calls(adi, p, plan, 1)
        b = _run_calls(adi, p, plan, 0)
        assert_parity(a, b, tol=1e-13, what=str(between[0][0]))


def test_carry_batch_point_sources(adi):
    """Carry with a batch of Ricker shots (per-grid point sources), split calls."""
    n, B = 1601, 2
    probs = [ricker_problem(n, shot=s, nshots=8, method=MFD, steps=8, f0=20.0, t0=0.05) for s in range(B)]
    p0 = probs[0]
    outs = []
    for carry, plan in ((1, [3, 2, 3]), (0, [8])):
        s = adi.AdiSolver(n, n, p0.h, p0.dt, 1.0, MFD, batch=B)
        s.set_param(adi.ADI_CARRY, carry)
        s.set_fields(np.stack([p.U for p in probs]), np.stack([p.V for p in probs]),
                     np.stack([p.W for p in probs]))
        s.set_point_sources([p.src[0] for p in probs], [p.src[1] for p in probs], p0.gf)
        for k in plan:
            s.step(k)
        outs.append(s.get_fields())
        s.close()
    assert np.abs(outs[1][0]).max() > 0
    assert_parity(outs[0], outs[1], tol=1e-13)


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n", [1601, 2101])
def test_async_store_knob_bitwise(adi, method, n):
    """ADI_ASYNC_STORE (bulk copies of X', TMA tensor stores of S'^T) changes how the outputs
    leave the tile, not their values: bitwise equal to the thread stores, split calls."""
    p = random_problem(method, n, seed=n + 11, steps=4)
    outs = []
    for v in (0, 1):
        s = adi.AdiSolver.from_problem(p)
        s.set_param(adi.ADI_ASYNC_STORE, v)
        s.step(1)
        s.step(3)
        outs.append(s.get_fields())
        s.close()
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def _short_run(adi, p, steps, warp, split=None, batch_probs=None):
    s = adi.AdiSolver.from_problem(p)
    s.set_param(adi.ADI_THREAD_LINES, 1)
    s.set_param(adi.ADI_WARP_LINES, warp)
    for k in (split or [steps]):
        s.step(k)
    out = s.get_fields()
    s.close()
    return out


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("nx,ny", [(9, 9), (17, 33), (41, 41), (61, 61), (41, 9), (9, 61), (62, 40),
                                   (63, 63), (81, 81), (130, 97), (161, 161), (321, 257), (383, 40),
                                   (384, 40)])
def test_warp_kernels_parity(adi, method, nx, ny):
    """Warp-per-line kernels (adi_warp.cuh): lines of up to 384 stored
    positions (2 .. 12 per lane, the instantiation edges 62/63 and 382/383 cells; 383 cells
    back on the tiles), random state, dense source, boundary data, split calls (prologue
    twice), against the oracle, and against the thread-per-line (or, where those do not
    fit, the tile) kernels to rounding (same LU recurrences, reassociated into warp scans)."""
    steps = 5
    p = random_problem(method, nx, ny=ny, seed=3 * nx + ny, steps=steps)
    w = _short_run(adi, p, steps, 1, split=[2, 3])
    assert_parity(w, run_oracle(p, steps), what=f"warp {nx}x{ny}")
    t = _short_run(adi, p, steps, 0, split=[2, 3])
    for name, a, b in zip("UVW", w, t):
        d = np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)
        assert d <= 1e-13, (name, d)


def test_warp_kernels_batch_points(adi):
    """A batch of point-source grids on the warp kernels (41^2, MFD and CFD)."""
    for method in (CFD, MFD):
        n, B, steps = 41, 3, 6
        probs = [random_problem(method, n, seed=60 + k, steps=steps, source=False) for k in range(B)]
        gf = np.random.default_rng(6).standard_normal(2 * steps + 1)
        for k, p in enumerate(probs):
            p.src = (5 + 7 * k, 30 - 9 * k)
            p.gf = gf
        p0 = probs[0]
        s = adi.AdiSolver(n, n, p0.h, p0.dt, p0.c, method, batch=B, K=p0.K)
        s.set_param(adi.ADI_THREAD_LINES, 1)
        s.set_fields(np.stack([p.U for p in probs]), np.stack([p.V for p in probs]), np.stack([p.W for p in probs]))
        s.set_point_sources([p.src[0] for p in probs], [p.src[1] for p in probs], gf)
        s.set_boundary(p0.edges, p0.gb)
        s.step(steps)
        got = s.get_fields()
        s.close()
        for k, p in enumerate(probs):
            q = p
            q.edges, q.gb = p0.edges, p0.gb
            assert_parity([x[k] for x in got], run_oracle(q, steps), what=f"warp batch {k} m{method}")


@pytest.mark.parametrize("method,n,graph", [(CFD, 41, 1), (MFD, 301, 0), (CFD, 1601, 0)])
def test_step_index_restart_bitwise(adi, method, n, graph):
    """ADI_STEP_INDEX with adi_set_fields restarts a run: a second call from the initial state
    at time level 0 reproduces the first call bitwise (graph replay, carried explicit half
    dropped, tables re-read from step 0)."""
    steps = 3
    p = random_problem(method, n, seed=n + 5, steps=steps)
    s = adi.AdiSolver.from_problem(p)
    s.set_param(adi.ADI_GRAPH, graph)
    s.step(steps)
    a = s.get_fields()
    s.set_fields(p.U, p.V, p.W)
    s.set_param(adi.ADI_STEP_INDEX, 0)
    s.step(steps)
    b = s.get_fields()
    with pytest.raises(adi.AdiError):
        s.set_param(adi.ADI_STEP_INDEX, -1)
    s.close()
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("nx,ny", [(4096, 41), (41, 4096), (3000, 77), (2101, 66), (4096, 4096)])
def test_frag_tiles_bitwise(adi, nx, ny):
    """ADI_FRAG_TILES: MFD lines whose tile plan leaves a short middle gap
    (4096 positions: 4 lean tiles + a 168-position fragment; 3000: 3 + 40) run the gap as
    8-chunk fragments packed 4 lines per warp.  The MFD halos are exact; positions owned by
    a line-end tile in one plan and an interior tile in the other differ only in the
    epilogue's rounding order, so max-norm <= 1e-14; split calls, and the
    oracle agrees."""
    steps = 2 if nx * ny > 1e6 else 3
    p = random_problem(MFD, nx, ny=ny, seed=nx + 7 * ny, steps=steps)
    outs = []
    for v in (1, 0):
        s = adi.AdiSolver.from_problem(p)
        s.set_param(adi.ADI_FRAG_TILES, v)
        s.step(1)
        s.step(steps - 1)
        outs.append(s.get_fields())
        s.close()
    for name, a, b in zip("UVW", *outs):
        d = np.abs(a - b).max() / np.abs(b).max()
        assert d <= 1e-14, (name, d)
    if nx * ny < 1e6:
        assert_parity(outs[0], run_oracle(p, steps), what=f"frag {nx}x{ny}")


def test_frag_tiles_batch_points(adi):
    """Fragment tiles with a batch of point-source grids (the config-5 launch shape, reduced),
    a source inside a fragment and one inside a lean tile; the standard plan to rounding."""
    n, B, steps = 4096, 3, 3
    probs = [random_problem(MFD, n, ny=40, seed=80 + k, steps=steps, source=False, boundary=False)
             for k in range(B)]
    gf = np.random.default_rng(8).standard_normal(2 * steps + 1)
    srcs = [(2000, 17), (500, 30), (2100, 3)]    # (x in the 4096 line's middle fragment: 1964..2131)
    outs = []
    for v in (1, 0):
        s = adi.AdiSolver(n, 40, probs[0].h, probs[0].dt, 1.0, MFD, batch=B)
        s.set_param(adi.ADI_FRAG_TILES, v)
        s.set_fields(np.stack([p.U for p in probs]), np.stack([p.V for p in probs]), np.stack([p.W for p in probs]))
        s.set_point_sources([a for a, _ in srcs], [b for _, b in srcs], gf)
        s.step(steps)
        outs.append(s.get_fields())
        s.close()
    for name, a, b in zip("UVW", *outs):
        d = np.abs(a - b).max() / np.abs(b).max()
        assert d <= 1e-14, (name, d)
    for k, p in enumerate(probs):
        p.src = srcs[k]
        p.gf = gf
        assert_parity([x[k] for x in outs[0]], run_oracle(p, steps), what=f"frag batch {k}")
