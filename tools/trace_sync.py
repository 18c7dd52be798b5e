"""Are the line kernel's tiles phase-synchronized?  Per-tile trace (adi_set_trace) of
one ADI-rows launch at 16384^2; prints the number of tiles in each phase (load / ops /
store) on a 1 us grid over a 120 us window mid-kernel, and the phase intervals of the
tiles of one SM."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2006_07583_b200 as adi
from adi_inputs import CFD, MFD, MMS, mms_problem

if os.environ.get("ADI_LIB"):   # a build variant (tools/build_variant.sh)
    adi.LIB_PATH = os.environ["ADI_LIB"]

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
meth = CFD if (len(sys.argv) < 3 or sys.argv[2] == "cfd") else MFD
cap = 1 << 20
buf = torch.zeros(8 * cap, dtype=torch.int64, device="cuda")
p = mms_problem(meth, n, MMS(), steps=8)
s = adi.AdiSolver.from_problem(p, stream=torch.cuda.current_stream().cuda_stream)
s.step(1)
adi.adi_set_trace(s.handle, buf, cap, 1)
s.step(1)
torch.cuda.synchronize()
adi.adi_set_trace(s.handle, None, 0, 0)
r = buf.view(cap, 8).cpu().numpy()
r = r[r[:, 5] > 0]
t0 = r[:, 2].min()
a, b, c, d = ((r[:, k] - t0) / 1e3 for k in (2, 3, 4, 5))
span = d.max()
e = (r[:, 6] - t0) / 1e3   # after the CTA barrier that precedes the stores
print(f"tiles {len(r)} span {span:.1f} us; mean load {np.mean(b-a):.2f} ops {np.mean(c-b):.2f} store {np.mean(d-c):.2f}"
      f" (barrier {np.mean(e-c):.2f} + issue {np.mean(d-e):.2f}); resident {((d - a).sum() / span):.0f}")
if os.environ.get("BRIEF"):
    sys.exit(0)
mid = span / 2
for t in np.arange(mid - 60, mid + 60, 1.0):
    nl = int(((a <= t) & (t < b)).sum()); no = int(((b <= t) & (t < c)).sum()); ns = int(((c <= t) & (t < d)).sum())
    print(f"t={t:8.1f} load {nl:4d} ops {no:4d} store {ns:4d}  " + "L" * (nl // 8) + "o" * (no // 8) + "s" * (ns // 8))
sm = r[:, 1]
one = np.where(sm == sm[len(sm) // 2])[0]
one = one[np.argsort(a[one])]
print("one SM:", sm[len(sm) // 2])
for i in one:
    if mid - 80 < a[i] < mid + 80:
        print(f"  tile {r[i,0]:7d} load {a[i]:8.1f}-{b[i]:8.1f} ops -{c[i]:8.1f} store -{d[i]:8.1f}")
