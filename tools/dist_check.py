"""Two-process check of the Python band driver (paper_2006_07583_b200/dist.py: BandSolver +
TorchDistTransport over torch.distributed) under torchrun, both ranks on device 0 with the
gloo backend: the halo messages are host-staged, so no rank's kernel ever waits on another's
(B200_PROFILING.md).  Rank 0 gathers the bands and prints the parity against the oracle.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/dist_check.py METHOD N STEPS
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import paper_2006_07583_b200 as adi
from paper_2006_07583_b200 import dist as adist
from adi_inputs import random_problem

method, n, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
p = random_problem(method, n, seed=50 + n, steps=steps)
stream = torch.cuda.current_stream()
s = adi.AdiSolver.from_problem(p, stream=stream.cuda_stream)
y0, y1, halo, npos = adi.adi_band_info(s.handle)
bs = adist.BandSolver(s, rank, world, adist.band_partition(npos, world, halo))
tr = adist.TorchDistTransport(rank, world)
adist.step_distributed(bs, tr, 1)
adist.step_distributed(bs, tr, steps - 1)   # two calls: the call-start U / W̄ exchange too
torch.cuda.synchronize()
mine = s.get_fields()
parts = [None] * world
dist.all_gather_object(parts, (mine, (bs.y0, bs.y1)))
if rank == 0:
    import oracle
    from parity import check
    got = adist.gather_bands([x[0] for x in parts], [x[1] for x in parts])
    o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=steps, **p.oracle_kwargs())
    for name, a, b in zip("UVW", got, o):
        check(a, b, name=name, what="torchrun 2 ranks")
    print("DIST_CHECK_OK", method, n, steps)
dist.barrier()
dist.destroy_process_group()
