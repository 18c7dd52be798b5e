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


# ---- adi_create_dist_local: the in-library exchange (adi_create_dist's code path with a
# loopback transport), band-local memory, the column sweep overlapping the transfer ----
def _dist_local(adi, p, world, **kw):
    hs = adi.adi_create_dist_local(p.nx, p.ny, p.h, p.dt, p.c, p.method, kw.get("batch", 1), world)
    ss = [adi.AdiSolver.adopt(h, p.nx, p.ny, p.h, p.dt, p.c, p.method, batch=kw.get("batch", 1), K=p.K)
          for h in hs]
    return hs, ss


def _gather_local(adi, ss, method, nx, ny, batch=1):
    """Each rank's band rows (adi_get_fields of a band writes only those) into one grid."""
    from adi_inputs import shapes
    from paper_2006_07583_b200 import dist
    parts = []
    bands = []
    for s in ss:
        out = [np.zeros(((batch,) if batch > 1 else ()) + sh) for sh in shapes(method, nx, ny)]
        adi.adi_get_fields(s.handle, *out)
        parts.append(out)
        y0, y1, _, _ = adi.adi_band_info(s.handle)
        bands.append((y0, y1))
    return dist.gather_bands(parts, bands)


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n,world,split", [(301, 2, [3]), (1601, 4, [1, 2]), (2101, 8, [2]), (4097, 3, [1, 1])])
def test_dist_local_equals_single_and_oracle(adi, method, n, world, split):
    """adi_create_dist_local + adi_step_dist_local (several calls: the kind-1 U/W̄ exchange
    too) against one plain handle and the oracle, rel L2 and max-norm."""
    steps = sum(split)
    p = random_problem(method, n, seed=n + 3 * world, steps=steps)
    hs, ss = _dist_local(adi, p, world)
    for s in ss:
        s.set_fields(p.U, p.V, p.W)
        s.set_source(p.phi, None, p.gf)
        s.set_boundary(p.edges, p.gb)
    for k in split:
        adi.adi_step_dist_local(hs, k)
    got = _gather_local(adi, ss, method, p.nx, p.ny)
    s1 = adi.AdiSolver.from_problem(p)
    s1.step(steps)
    ref = s1.get_fields()
    s1.close()
    o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=steps, **p.oracle_kwargs())
    for name, a, b, c in zip("UVW", got, ref, o):
        check(a, b, tol=1e-13, name=name, what="dist_local vs one handle")
        check(a, c, name=name, what="dist_local vs oracle")
    for s in ss:
        with pytest.raises(adi.AdiError):
            adi.adi_step(s.handle, 1)            # ranks of a local group step together
        with pytest.raises(adi.AdiError):
            adi.adi_set_band(s.handle, 0, 64)    # the band of a dist handle is fixed
    for s in ss:
        s.close()


def test_dist_local_media_batch_points(adi):
    """Media, a batch of point-source shots and the dist-local exchange together."""
    n, world, B, steps = 1601, 3, 2, 3
    probs = [ricker_problem(n, shot=s, nshots=4, steps=steps, f0=20.0, t0=0.05) for s in range(B)]
    p0 = probs[0]
    rng = np.random.default_rng(5)
    med = [rng.uniform(0.6, 1.0, a.shape).astype(np.float32) for a in (p0.U, p0.V, p0.W)]
    hs, ss = _dist_local(adi, p0, world, batch=B)
    U = np.stack([p.U for p in probs]); V = np.stack([p.V for p in probs]); W = np.stack([p.W for p in probs])
    rng2 = np.random.default_rng(6)
    U = U + rng2.standard_normal(U.shape)   # a nonzero start (the sources are weak early)
    for s in ss:
        s.set_fields(U, V, W)
        s.set_point_sources([p.src[0] for p in probs], [p.src[1] for p in probs], p0.gf)
        s.set_media(*med)
    adi.adi_step_dist_local(hs, steps)
    got = _gather_local(adi, ss, MFD, n, n, batch=B)
    for b, p in enumerate(probs):
        o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, U[b], p.V, p.W, nsteps=steps,
                       src=p.src, gf=p.gf, kappa=med[0], rinv_v=med[1], rinv_w=med[2])
        for name, a, c in zip("UVW", got, o):
            check(a[b], c, name=name, what=f"dist_local media shot {b}")
    for s in ss:
        s.close()


def test_dist_memory_scales_with_bands(adi):
    """Per-rank device memory of a band-local handle (adi_get_stats device_bytes): at P = 8
    each rank holds its band + halo rows, <= 1/6 of the P = 1 handle; adi_set_band on a
    plain handle re-lays its arrays out the same way."""
    n = 8193
    h = 1.0 / (n - 1)
    for method in (CFD, MFD):
        hs1 = adi.adi_create_dist_local(n, n, h, 0.5 * h, 1.0, method, 1, 1)
        b1 = adi.adi_get_stats(hs1[0])["device_bytes"]
        adi.adi_destroy(hs1[0])
        hs8 = adi.adi_create_dist_local(n, n, h, 0.5 * h, 1.0, method, 1, 8)
        b8 = [adi.adi_get_stats(x)["device_bytes"] for x in hs8]
        for x in hs8:
            adi.adi_destroy(x)
        assert max(b8) <= b1 / 6, (method, b1, b8)
        s = adi.AdiSolver(n, n, h, 0.5 * h, 1.0, method)
        full = s.stats()["device_bytes"]
        y0, y1, halo, npos = adi.adi_band_info(s.handle)
        adi.adi_set_band(s.handle, npos // 2, npos // 2 + 1024)
        assert s.stats()["device_bytes"] <= full / 6
        s.close()


# ---- ADI_DIST_TRANSPOSE: the north_star's all-to-all decomposition (loopback transport) ----
def _gather_dist(adi, ss, method, nx, ny, batch=1):
    """Assemble a grid from the ranks' owned parts (adi_dist_info): U and W̄ by columns and
    V̄ by rows in transpose mode; U, V̄, W̄ by rows in halo mode."""
    from adi_inputs import shapes
    su, sv, sw = shapes(method, nx, ny)
    pre = (batch,) if batch > 1 else ()
    U, V, W = np.zeros(pre + su), np.zeros(pre + sv), np.zeros(pre + sw)
    off = 1
    for s in ss:
        parts = [np.zeros(pre + sh) for sh in (su, sv, sw)]
        adi.adi_get_fields(s.handle, *parts)
        mode, r0, r1, c0, c1 = adi.adi_dist_info(s.handle)
        npy, npx = ny, nx
        re = None if r1 >= npy else r1
        ce = None if c1 >= npx else c1
        V[..., max(r0 - off, 0):(None if re is None else max(re - off, 0)), :] = \
            parts[1][..., max(r0 - off, 0):(None if re is None else max(re - off, 0)), :]
        if mode == adi.ADI_DIST_TRANSPOSE:
            U[..., :, c0:ce] = parts[0][..., :, c0:ce]
            W[..., :, max(c0 - off, 0):(None if ce is None else max(ce - off, 0))] = \
                parts[2][..., :, max(c0 - off, 0):(None if ce is None else max(ce - off, 0))]
        else:
            U[..., r0:re, :] = parts[0][..., r0:re, :]
            W[..., r0:re, :] = parts[2][..., r0:re, :]
    return U, V, W


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n,world,split", [(301, 2, [3]), (1601, 4, [1, 2]), (2101, 8, [2]), (517, 3, [1])])
def test_dist_local_transpose_equals_single_and_oracle(adi, method, n, world, split):
    """ADI_DIST_TRANSPOSE through adi_create_dist_local_ex: rows and columns owned by
    different ranks, S moved by the all-to-all; against one handle and the oracle."""
    steps = sum(split)
    p = random_problem(method, n, seed=7 * n + world, steps=steps)
    hs = adi.adi_create_dist_local(p.nx, p.ny, p.h, p.dt, p.c, method, 1, world, adi.ADI_DIST_TRANSPOSE)
    ss = [adi.AdiSolver.adopt(h, p.nx, p.ny, p.h, p.dt, p.c, method, K=p.K) for h in hs]
    for s in ss:
        s.set_fields(p.U, p.V, p.W)
        s.set_source(p.phi, None, p.gf)
        s.set_boundary(p.edges, p.gb)
    for k in split:
        adi.adi_step_dist_local(hs, k)
    got = _gather_dist(adi, ss, method, p.nx, p.ny)
    s1 = adi.AdiSolver.from_problem(p)
    s1.step(steps)
    ref = s1.get_fields()
    s1.close()
    o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=steps, **p.oracle_kwargs())
    for name, a, b, c in zip("UVW", got, ref, o):
        check(a, b, tol=1e-13, name=name, what="transpose vs one handle")
        check(a, c, name=name, what="transpose vs oracle")
    for s in ss:
        with pytest.raises(adi.AdiError):
            adi.adi_halo_bytes(s.handle, 0, 0)
        s.close()


def test_dist_local_transpose_batch_points_and_memory(adi):
    """A batch of point-source shots in the transpose decomposition; per-rank memory at
    P = 8 is a small fraction of the P = 1 handle."""
    n, world, B, steps = 1601, 4, 2, 3
    probs = [ricker_problem(n, shot=s, nshots=4, steps=steps, f0=20.0, t0=0.05) for s in range(B)]
    p0 = probs[0]
    rng = np.random.default_rng(8)
    U = np.stack([p.U for p in probs]) + rng.standard_normal((B,) + p0.U.shape)
    V = np.stack([p.V for p in probs]); W = np.stack([p.W for p in probs])
    hs = adi.adi_create_dist_local(n, n, p0.h, p0.dt, 1.0, MFD, B, world, adi.ADI_DIST_TRANSPOSE)
    ss = [adi.AdiSolver.adopt(h, n, n, p0.h, p0.dt, 1.0, MFD, batch=B) for h in hs]
    for s in ss:
        s.set_fields(U, V, W)
        s.set_point_sources([p.src[0] for p in probs], [p.src[1] for p in probs], p0.gf)
    adi.adi_step_dist_local(hs, steps)
    got = _gather_dist(adi, ss, MFD, n, n, batch=B)
    for b, p in enumerate(probs):
        o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, U[b], p.V, p.W, nsteps=steps, src=p.src, gf=p.gf)
        for name, a, c in zip("UVW", got, o):
            check(a[b], c, name=name, what=f"transpose shot {b}")
    for s in ss:
        s.close()
    m = 8193
    h = 1.0 / (m - 1)
    one = adi.adi_create_dist_local(m, m, h, 0.5 * h, 1.0, CFD, 1, 1)
    b1 = adi.adi_get_stats(one[0])["device_bytes"]
    adi.adi_destroy(one[0])
    eight = adi.adi_create_dist_local(m, m, h, 0.5 * h, 1.0, CFD, 1, 8, adi.ADI_DIST_TRANSPOSE)
    b8 = [adi.adi_get_stats(x)["device_bytes"] for x in eight]
    for x in eight:
        adi.adi_destroy(x)
    assert max(b8) <= b1 / 5, (b1, b8)


@pytest.mark.parametrize("method", [CFD, MFD])
def test_torchrun_two_ranks_python_band_driver(adi, method):
    """Two processes under torchrun (gloo, both on device 0, host-staged halo messages: no
    kernel waits on another rank): the Python band driver (dist.py) against the oracle."""
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ, PYTHONPATH=os.path.join(root, "tests") + os.pathsep + root)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), "tools/dist_check.py",
                          str(method), "1601", "3"], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "DIST_CHECK_OK" in out.stdout


def _run_transpose(adi, p, world, fused, split, batch=1, setup=None):
    hs = adi.adi_create_dist_local(p.nx, p.ny, p.h, p.dt, p.c, p.method, batch, world, adi.ADI_DIST_TRANSPOSE)
    ss = [adi.AdiSolver.adopt(h, p.nx, p.ny, p.h, p.dt, p.c, p.method, K=p.K, batch=batch) for h in hs]
    for s in ss:
        s.set_param(adi.ADI_DIST_FUSED, fused)
        if setup:
            setup(s)
        else:
            s.set_fields(p.U, p.V, p.W)
            s.set_source(p.phi, None, p.gf)
            s.set_boundary(p.edges, p.gb)
    for k in split:
        adi.adi_step_dist_local(hs, k)
    got = _gather_dist(adi, ss, p.method, p.nx, p.ny, batch=batch)
    for s in ss:
        s.close()
    return got


@pytest.mark.parametrize("method", [CFD, MFD])
@pytest.mark.parametrize("n,world,split", [(301, 2, [3]), (1601, 4, [1, 2]), (2101, 8, [2]), (517, 3, [2, 1])])
def test_dist_local_transpose_fused_bitwise(adi, method, n, world, split):
    """ADI_DIST_FUSED: the row / column kernels store S' straight into the
    owning rank's array and the all-to-all becomes a barrier -- bitwise the fields of the
    all-to-all, split calls (prologue after set_fields and between calls), and the oracle."""
    steps = sum(split)
    p = random_problem(method, n, seed=5 * n + world, steps=steps)
    fz = _run_transpose(adi, p, world, 1, split)
    a2a = _run_transpose(adi, p, world, 0, split)
    for a, b in zip(fz, a2a):
        assert np.array_equal(a, b)
    o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=steps, **p.oracle_kwargs())
    for name, a, c in zip("UVW", fz, o):
        check(a, c, name=name, what="fused transpose vs oracle")


def test_dist_local_transpose_fused_batch_points(adi):
    """Fused transpose with a batch of point-source grids (per-grid peer strides)."""
    n, world, B, steps = 1601, 4, 3, 3
    probs = [ricker_problem(n, shot=s, nshots=4, steps=steps, f0=20.0, t0=0.05) for s in range(B)]
    p0 = probs[0]
    rng = np.random.default_rng(9)
    U = np.stack([p.U for p in probs]) + rng.standard_normal((B,) + p0.U.shape)
    V = np.stack([p.V for p in probs]); W = np.stack([p.W for p in probs])

    def setup(s):
        s.set_fields(U, V, W)
        s.set_point_sources([p.src[0] for p in probs], [p.src[1] for p in probs], p0.gf)
    fz = _run_transpose(adi, p0, world, 1, [steps], batch=B, setup=setup)
    a2a = _run_transpose(adi, p0, world, 0, [steps], batch=B, setup=setup)
    for a, b in zip(fz, a2a):
        assert np.array_equal(a, b)
    for b, p in enumerate(probs):
        o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, U[b], p.V, p.W, nsteps=steps, src=p.src, gf=p.gf)
        for name, a, c in zip("UVW", fz, o):
            check(a[b], c, name=name, what=f"fused transpose shot {b}")


def test_dist_fused_param_validation(adi):
    """ADI_DIST_FUSED exists only on transpose-mode ranks with a peer table."""
    p = random_problem(MFD, 129, seed=3, steps=1)
    hs = adi.adi_create_dist_local(p.nx, p.ny, p.h, p.dt, p.c, MFD, 1, 2)   # halo mode
    for h in hs:
        with pytest.raises(adi.AdiError):
            adi.adi_set_param(h, adi.ADI_DIST_FUSED, 1)
        adi.adi_set_param(h, adi.ADI_DIST_FUSED, 0)
        adi.adi_destroy(h)
    s = adi.AdiSolver.from_problem(p)
    with pytest.raises(adi.AdiError):
        s.set_param(adi.ADI_DIST_FUSED, 1)
    with pytest.raises(adi.AdiError):
        s.set_param(adi.ADI_DIST_FUSED, 2)
    s.close()


def test_dist_local_transpose_fused_with_fragment_plan(adi):
    """MFD lines with a fragment plan (4096 positions) in the transpose
    decomposition: the PACK fragments store their S' into the owning ranks' arrays too, so
    fused and all-to-all agree bitwise, and one handle to rounding."""
    p = random_problem(MFD, 4096, ny=200, seed=21, steps=3)
    fz = _run_transpose(adi, p, 2, 1, [1, 2])
    a2a = _run_transpose(adi, p, 2, 0, [1, 2])
    s = adi.AdiSolver.from_problem(p)
    s.step(1)
    s.step(2)
    one = s.get_fields()
    s.close()
    for name, a, b, c in zip("UVW", fz, a2a, one):
        assert np.array_equal(a, b), name
        assert np.abs(a - c).max() <= 1e-14 * np.abs(c).max(), name
