"""Tile timeline of the line kernels (adi_set_trace): phase durations, SM
occupancy over the kernel span and how many tiles are in each phase at once."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2006_07583_b200 as adi

if os.environ.get("ADI_LIB"):   # a build with -DADI_TILE_TRACE=1 (tools/build_variant.sh)
    adi.LIB_PATH = os.environ["ADI_LIB"]
from adi_inputs import CFD, MFD, MMS, mms_problem

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/trace"
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
KIND = {"row": 1, "col": 2, "final": 3, "prologue": 0}
cap = 1 << 20
buf = torch.zeros(8 * cap, dtype=torch.int64, device="cuda")
for method in (MFD, CFD):
    mname = ("CFD", "MFD")[method]
    p = mms_problem(method, n, MMS(), steps=40)
    s = adi.AdiSolver.from_problem(p, stream=torch.cuda.current_stream().cuda_stream)
    if True:
        for kname in ("row", "col", "final", "prologue"):
            s.set_fields(p.U, p.V, p.W)
            s.step(1)
            buf.zero_()
            adi.adi_set_trace(s.handle, buf, cap, KIND[kname])
            s.step(2)
            torch.cuda.synchronize()
            adi.adi_set_trace(s.handle, None, 0, 0)
            s.m = 0
            r = buf.view(cap, 8).cpu().numpy()
            r = r[r[:, 5] > 0]
            np.save(f"{out}_{mname}_{kname}.npy", r)
            t0 = r[:, 2].min()
            a, b_, c_, d = (r[:, 2] - t0) / 1e3, (r[:, 3] - t0) / 1e3, (r[:, 4] - t0) / 1e3, (r[:, 5] - t0) / 1e3
            span = d.max()
            busy = (d - a).sum()
            nsm = len(np.unique(r[:, 1]))
            # concurrency per phase sampled on a 0.5 us grid
            grid = np.arange(0, span, 0.5)
            def conc(lo, hi):
                lo_i = np.searchsorted(grid, lo); hi_i = np.searchsorted(grid, hi)
                cnt = np.zeros(len(grid) + 1); np.add.at(cnt, lo_i, 1); np.add.at(cnt, hi_i, -1)
                return np.cumsum(cnt)[:-1]
            cl, co, cs = conc(a, b_), conc(b_, c_), conc(c_, d)
            mid = slice(len(grid) // 10, 9 * len(grid) // 10)
            print(f"{mname} {kname:8s} tiles={len(r)} span={span/1e3:.3f} ms "
                  f"tile us: load {np.mean(b_-a):.1f} ops {np.mean(c_-b_):.1f} store {np.mean(d-c_):.1f} "
                  f"total {np.mean(d-a):.1f} | resident avg {busy/span:.0f} ({busy/span/nsm:.2f}/SM) | "
                  f"in phase (mid 80%): load {cl[mid].mean():.0f} ops {co[mid].mean():.0f} store {cs[mid].mean():.0f}",
                  flush=True)
