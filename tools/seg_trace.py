"""Per-segment tile durations of one line-kernel launch (adi_set_trace)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2006_07583_b200 as adi

if os.environ.get("ADI_LIB"):   # a build with -DADI_TILE_TRACE=1 (tools/build_variant.sh)
    adi.LIB_PATH = os.environ["ADI_LIB"]
from adi_inputs import CFD, MFD, MMS, mms_problem

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
kind = {"row": 1, "col": 2, "final": 3, "prologue": 0}[sys.argv[2] if len(sys.argv) > 2 else "row"]
cap = 1 << 20
buf = torch.zeros(8 * cap, dtype=torch.int64, device="cuda")
for method in (MFD, CFD):
    p = mms_problem(method, n, MMS(), steps=40)
    s = adi.AdiSolver.from_problem(p, stream=torch.cuda.current_stream().cuda_stream)
    s.set_fields(p.U, p.V, p.W)
    s.step(1)
    adi.adi_set_trace(s.handle, buf, cap, kind)
    s.step(2)
    torch.cuda.synchronize()
    adi.adi_set_trace(s.handle, None, 0, 0)
    r = buf.view(cap, 8).cpu().numpy()
    r = r[r[:, 5] > 0]
    gx = (n - 1 + 3) // 4 if True else 0
    tile = r[:, 0]
    # grid x = line groups: infer from the max tile id and the segment count
    ntiles = tile.max() + 1
    nseg = None
    for cand in range(1, 64):
        if ntiles % cand == 0 and ntiles // cand in (n // 4, (n - 1) // 4 + 1, (n - 2) // 4 + 1, n // 4 + 1):
            nseg = cand
            break
    gX = ntiles // nseg
    seg = (tile // gX) % nseg
    tot = (r[:, 5] - r[:, 2]) / 1e3
    ops = (r[:, 4] - r[:, 3]) / 1e3
    print(("CFD", "MFD")[method], f"segments {nseg}, line groups {gX}")
    for k in range(nseg):
        m = seg == k
        print(f"  seg {k:2d}: tiles {m.sum():5d} total {tot[m].mean():6.1f} us  ops {ops[m].mean():6.1f} us")
