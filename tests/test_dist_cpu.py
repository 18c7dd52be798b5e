"""CPU coverage of the multi-GPU path (gloo, world size 2).

* band_partition: bands tile the line, are 4-aligned and at least a halo thick.
* TorchDistTransport: the exact point-to-point exchange used with NCCL, run
  on gloo between two processes.
* The band claim behind the halo exchange: a rank that
  holds correct inputs only on its band +- halo (garbage elsewhere) and
  receives the halo from its neighbour reproduces, on its band, the oracle's
  full-line column half-step (a6 + epilogue) to round-off."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from adi_inputs import CFD, MFD
from paper_2006_07583_b200.dist import (HIGH, LOW, TorchDistTransport, band_partition,
                                        neighbours)

def shipped_halo(method):
    """The halo the library's band plan uses (adi_plan_halo, host logic: no GPU needed)."""
    import paper_2006_07583_b200 as adi
    return adi.adi_plan_halo(method)


@pytest.mark.parametrize("npos,world,halo", [(301, 2, 64), (1602, 4, 64), (16384, 8, 64),
                                             (9, 1, 64), (258, 3, 32)])
def test_band_partition(npos, world, halo):
    bands = band_partition(npos, world, halo)
    assert bands[0][0] == 0 and bands[-1][1] == npos
    for (a, b), (c, d) in zip(bands, bands[1:]):
        assert b == c and (c - 1) % 4 == 0
    assert all(b - a >= halo or world == 1 for a, b in bands)


def test_band_partition_rejects_thin_bands():
    with pytest.raises(ValueError):
        band_partition(100, 4, 64)


def _half_step_column(method, n, h, K, alpha, beta, s, w0, gB, gT, fsrc):
    """Oracle column half-step of one line: K sweeps (eq. 9) then the fused
    epilogue S' = u - alpha D̄(w) + dt/2 F, X' = w - beta D([gB,u,gT])."""
    u, w = oracle.stage_line(method, n, h, K, alpha, beta, s, w0, gB, gT)
    Sp = u - alpha * oracle.apply_Dbar(method, n, h, w) + fsrc
    ub = np.concatenate([[gB], u, [gT]])
    Xp = w - beta * oracle.apply_D(method, n, h, ub)
    return Sp, Xp


def _worker(rank, world, port, method, n, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h = 1.0 / n
        dt = (0.91 if method == CFD else 0.81) * h
        alpha = beta = dt / 2
        K = 8
        rng = np.random.default_rng(42)              # same full data on every rank
        nu = n - 1 if method == CFD else n
        s_full = rng.standard_normal(nu)
        w_full = rng.standard_normal(n + 1)
        f_full = rng.standard_normal(nu) * dt / 2
        gB, gT = 0.3, -0.7
        Sref, Xref = _half_step_column(method, n, h, K, alpha, beta, s_full, w_full, gB, gT, f_full)
        # this rank's band of y positions and its halo
        halo = shipped_halo(method)
        bands = band_partition(n + 1, world, halo)
        y0, y1 = bands[rank]
        lo, hi = max(y0 - halo, 0), min(y1 + halo, n + 1)
        garb = np.random.default_rng(100 + rank)
        # local copies: correct only on the band, garbage elsewhere (u index = position - 1)
        s = garb.standard_normal(nu)
        w = garb.standard_normal(n + 1)
        s[max(y0 - 1, 0):max(y1 - 1, 0)] = s_full[max(y0 - 1, 0):max(y1 - 1, 0)]
        w[y0:y1] = w_full[y0:y1]
        # halo exchange through the transport: send my edge positions, receive the neighbour's
        tr = TorchDistTransport(rank, world)
        send, recv = {}, {}
        for side in neighbours(rank, world):
            a, b = (y0, min(y0 + halo, y1)) if side == LOW else (max(y1 - halo, y0), y1)
            msg = np.concatenate([w[a:b], [s[p - 1] if 1 <= p <= nu else 0.0 for p in range(a, b)]])
            send[side] = torch.tensor(msg)
            recv[side] = torch.zeros(2 * halo, dtype=torch.float64)
        tr.exchange(send, recv)
        for side, buf in recv.items():
            a, b = (lo, y0) if side == LOW else (y1, hi)
            v = buf.numpy()
            w[a:b] = v[:b - a]
            for k, p in enumerate(range(a, b)):
                if 1 <= p <= nu:
                    s[p - 1] = v[halo + k]
        f = f_full.copy()   # the source is static data every rank holds
        Sp, Xp = _half_step_column(method, n, h, K, alpha, beta, s, w, gB, gT, f)
        # compare on the band
        xs = slice(y0, y1)
        us = slice(max(y0 - 1, 0), min(max(y1 - 1, 0), nu))
        ex = np.abs(Xp[xs] - Xref[xs]).max() / np.abs(Xref).max()
        es = np.abs(Sp[us] - Sref[us]).max() / np.abs(Sref).max()
        # and the garbage really matters outside band+halo (the test is not vacuous)
        results[rank] = (ex, es, np.abs(Xp - Xref).max() / np.abs(Xref).max())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("method", [CFD, MFD])
def test_band_halo_exchange_gloo(method):
    world, n = 2, 400
    mgr = mp.Manager()
    results = mgr.dict()
    port = 29500 + 7 * method + os.getpid() % 500
    mp.spawn(_worker, args=(world, port, method, n, results), nprocs=world, join=True)
    assert shipped_halo(method) == (56 if method == CFD else 28)
    for r in range(world):
        ex, es, whole = results[r]
        assert ex < 1e-14 and es < 1e-14, (r, ex, es)
        assert whole > 1e-3   # outside the band the garbage changed the result
