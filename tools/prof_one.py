"""Minimal driver for ncu: one ADI call of `steps` steps on an n x n MMS grid
(argv[4] == "media": in the bench's heterogeneous medium, NEXT row f3)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_07583_b200 as adi
from adi_inputs import CFD, MFD
from bench import make_problem

method = {"cfd": CFD, "mfd": MFD, "cfd_full": 2}[sys.argv[1]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
media = len(sys.argv) > 4 and sys.argv[4] == "media"
p = make_problem(method, n, steps + 2, 8, media)
s = adi.AdiSolver.from_problem(p)
if method == 2:
    from bench import ABSORB_NB, ABSORB_A
    s.set_param(adi.ADI_ABSORB_WIDTH, ABSORB_NB)
    s.set_param(adi.ADI_ABSORB_RATE, ABSORB_A)
s.step(steps)
s.get_fields()
print("ok", sys.argv[1], n, steps, "media" if media else "")
