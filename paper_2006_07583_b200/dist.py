"""Multi-GPU band decomposition of one ADI grid.

Every sweep's lines are independent.  Rank r owns a band of y
positions:
- its row sweep handles the interior rows of the band;
- its column sweep outputs the band's positions and needs the carried field S2
  and the velocity W* in a halo of `halo` positions on each side.
The halo is exact to round-off because a half-step's domain of influence is
bounded.  One halo exchange per step (kind 0, after the row
sweep) plus one per call (kind 1, before the prologue) replaces the
all-to-all transpose of the north_star.

The arithmetic stays in libadi.so.  This module only moves the contiguous halo
messages that `adi_halo_pack` / `adi_halo_unpack` produce, over
torch.distributed (NCCL between GPUs, gloo on CPU) or between the handles of
an in-process group (single-GPU verification: ranks run one after another, no
rank ever waits on another).
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

HALO_SW = 0   # S2 and W* (after the row sweep)
HALO_UW = 1   # U and W̄ (before the prologue of a call)
LOW, HIGH = 0, 1


def band_partition(npos: int, world: int, halo: int, align: int = 4) -> List[Tuple[int, int]]:
    """Split y positions [0, npos) into `world` contiguous bands.

    Interior cuts b satisfy (b - 1) % align == 0, so each band's row sweep
    starts on a group of `align` lines (32-byte transposed writes).  Every band
    must be at least `halo` positions thick.
    """
    if world < 1:
        raise ValueError("world < 1")
    cuts = [0]
    for k in range(1, world):
        b = k * npos / world
        b = 1 + align * max(1, int(round((b - 1) / align)))
        cuts.append(b)
    cuts.append(npos)
    bands = [(cuts[i], cuts[i + 1]) for i in range(world)]
    for a, b in bands:
        if world > 1 and b - a < halo:
            raise ValueError(f"band {a}:{b} thinner than the halo {halo}")
    return bands


def neighbours(rank: int, world: int) -> Dict[int, int]:
    """side -> neighbour rank."""
    out = {}
    if rank > 0:
        out[LOW] = rank - 1
    if rank < world - 1:
        out[HIGH] = rank + 1
    return out


def opposite(side: int) -> int:
    return LOW if side == HIGH else HIGH


class TorchDistTransport:
    """Halo exchange with torch.distributed point-to-point (NCCL or gloo)."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group

    def exchange(self, send: Dict[int, "torch.Tensor"], recv: Dict[int, "torch.Tensor"]):
        import torch
        import torch.distributed as dist
        nb = neighbours(self.rank, self.world)
        if not nb:
            return
        staged = dist.get_backend(self.group) != "nccl" and any(t.is_cuda for t in send.values())
        if staged:   # gloo: host-staged messages (CPU tests, single-device functional checks)
            torch.cuda.current_stream().synchronize()
            snd = {k: v.cpu() for k, v in send.items()}
            rcv = {k: torch.empty_like(v, device="cpu") for k, v in recv.items()}
        else:
            snd, rcv = send, recv
        ops = []
        for side, peer in nb.items():
            ops.append(dist.P2POp(dist.isend, snd[side], peer, group=self.group))
            ops.append(dist.P2POp(dist.irecv, rcv[side], peer, group=self.group))
        for r in dist.batch_isend_irecv(ops):
            r.wait()
        if staged:
            for k in recv:
                recv[k].copy_(rcv[k])


class BandSolver:
    """One rank's share of a band-decomposed grid (wraps an AdiSolver)."""

    def __init__(self, solver, rank: int, world: int, bands: Sequence[Tuple[int, int]]):
        import torch
        from . import adi_band_info, adi_halo_bytes, adi_set_band
        self.s, self.rank, self.world = solver, rank, world
        y0, y1 = bands[rank]
        adi_set_band(solver.handle, y0, y1)
        self.y0, self.y1, self.halo, self.npos = adi_band_info(solver.handle)
        self.nb = neighbours(rank, world)
        self.bufs = {}
        for kind in (HALO_SW, HALO_UW):
            for side in self.nb:
                nbytes = adi_halo_bytes(solver.handle, kind, side)
                for d in ("send", "recv"):
                    self.bufs[(kind, side, d)] = torch.zeros(nbytes // 8, dtype=torch.float64,
                                                             device="cuda")
        self.fresh = True  # right after set_fields every rank holds the full state

    def pack(self, kind):
        from . import adi_halo_pack
        out = {}
        for side in self.nb:
            b = self.bufs[(kind, side, "send")]
            adi_halo_pack(self.s.handle, kind, side, b)
            out[side] = b
        return out

    def recv_buffers(self, kind):
        return {side: self.bufs[(kind, side, "recv")] for side in self.nb}

    def unpack(self, kind):
        from . import adi_halo_unpack
        for side in self.nb:
            adi_halo_unpack(self.s.handle, kind, side, self.bufs[(kind, side, "recv")])

    def set_fields(self, U, V, W):
        self.s.set_fields(U, V, W)
        self.fresh = True


def step_distributed(bs: BandSolver, transport, n: int):
    """adi_step(n) of one rank, with the halo exchanges in between (collective).

    The library must run on torch's current stream (AdiSolver(stream=...)) so
    that packing, the transport and unpacking are ordered."""
    from . import adi_step_begin, adi_step_cols, adi_step_end, adi_step_rows
    h = bs.s.handle
    if not bs.fresh:
        _exchange(bs, transport, HALO_UW)
    adi_step_begin(h, n)
    for _ in range(n):
        adi_step_rows(h)
        _exchange(bs, transport, HALO_SW)
        adi_step_cols(h)
    adi_step_end(h)
    bs.fresh = False


def _exchange(bs: BandSolver, transport, kind):
    send = bs.pack(kind)
    transport.exchange(send, bs.recv_buffers(kind))
    bs.unpack(kind)


class LocalGroup:
    """All ranks of a band decomposition in ONE process on one device.

    Verifies the decomposition on a single GPU: the ranks' kernels run one
    after another on one stream and messages are device copies, so no rank
    ever waits on another (B200_PROFILING.md)."""

    def __init__(self, solvers, bands):
        self.ranks = [BandSolver(s, r, len(solvers), bands) for r, s in enumerate(solvers)]

    def _exchange(self, kind):
        sends = [bs.pack(kind) for bs in self.ranks]
        for bs in self.ranks:
            for side, peer in bs.nb.items():
                bs.bufs[(kind, side, "recv")].copy_(sends[peer][opposite(side)])
        for bs in self.ranks:
            bs.unpack(kind)

    def step(self, n: int):
        from . import adi_step_begin, adi_step_cols, adi_step_end, adi_step_rows
        if not all(bs.fresh for bs in self.ranks):
            self._exchange(HALO_UW)
        for bs in self.ranks:
            adi_step_begin(bs.s.handle, n)
        for _ in range(n):
            for bs in self.ranks:
                adi_step_rows(bs.s.handle)
            self._exchange(HALO_SW)
            for bs in self.ranks:
                adi_step_cols(bs.s.handle)
        for bs in self.ranks:
            adi_step_end(bs.s.handle)
            bs.fresh = False

    def gather(self):
        """Assemble (U, V̄, W̄) from the bands (host arrays)."""
        return gather_bands([bs.s.get_fields() for bs in self.ranks], [(bs.y0, bs.y1) for bs in self.ranks])


def gather_bands(parts, bands):
    """Combine per-rank full-size (U, V̄, W̄) whose rows are valid on their band.

    U rows and W̄ rows are y positions; V̄ row j is y position j + 1."""
    U = parts[0][0].copy()
    V = parts[0][1].copy()
    W = parts[0][2].copy()
    last = len(bands) - 1
    for k, ((Ur, Vr, Wr), (y0, y1)) in enumerate(zip(parts, bands)):
        e = None if k == last else y1          # the last band also owns any rows above
        U[..., y0:e, :] = Ur[..., y0:e, :]
        W[..., y0:e, :] = Wr[..., y0:e, :]
        a = max(y0 - 1, 0)
        eb = None if k == last else max(y1 - 1, 0)
        V[..., a:eb, :] = Vr[..., a:eb, :]
    return U, V, W
