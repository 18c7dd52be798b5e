"""Minimal driver for ncu: one ADI call of `steps` steps on an n x n MMS grid."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_07583_b200 as adi
from adi_inputs import CFD, MFD, MMS, mms_problem

method = {"cfd": CFD, "mfd": MFD}[sys.argv[1]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
p = mms_problem(method, n, MMS(), steps=steps + 2)
s = adi.AdiSolver.from_problem(p)
s.step(steps)
s.get_fields()
print("ok", sys.argv[1], n, steps)
