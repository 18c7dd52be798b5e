"""Diagnostics: GPU-vs-oracle relative L2 per field as a function of step count,
next to the oracle's own sensitivity to a 1-ulp input perturbation."""
import math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_2006_07583_b200 as adi
from adi_inputs import CFD, MFD, MMS, mms_problem

def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)

T = 1 / math.sqrt(2)
for method, n, kw, checkpoints in ((MFD, 41, dict(t_sim=5 * T), [1, 10, 50, 100, 175]),
                                    (CFD, 41, dict(steps=200), [1, 10, 25, 50, 75, 100, 150, 200])):
    p = mms_problem(method, n, MMS(), **kw)
    s = adi.AdiSolver.from_problem(p)
    q = mms_problem(method, n, MMS(), **kw)
    q.U = q.U * (1 + 2.0 ** -52)
    done = 0
    for st in checkpoints:
        s.step(st - done)
        done = st
        g = s.get_fields()
        o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=st, **p.oracle_kwargs())
        o2 = oracle.run(q.method, q.nx, q.ny, q.h, q.dt, q.c, q.K, q.U, q.V, q.W, nsteps=st, **q.oracle_kwargs())
        print(("CFD", "MFD")[method], n, "steps", st,
              " gpu-vs-oracle " + " ".join(f"{nm}={rel(a, b):.2e}" for nm, a, b in zip("UVW", g, o)),
              " | oracle 1ulp-sensitivity " + " ".join(f"{nm}={rel(c, b):.2e}" for nm, c, b in zip("UVW", o2, o)),
              " | norms " + " ".join(f"{np.linalg.norm(b):.2e}" for b in o))
    s.close()
