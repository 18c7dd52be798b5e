import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2006_07583_b200 as adi
from adi_inputs import CFD, MFD, random_problem
try:
    from cuda.bindings import runtime as cudart
except Exception:
    from cuda import cudart
p = random_problem(MFD, 77, seed=11, steps=1)
s = adi.AdiSolver.from_problem(p); s.step(1); ref = s.get_fields(); s.close()
for flags, name in ((0, "blocking"), (1, "non-blocking")):
    err, st = cudart.cudaStreamCreateWithFlags(flags)
    res = []
    for _ in range(12):
        s = adi.AdiSolver.from_problem(p, stream=int(st)); s.step(1); o = s.get_fields(); s.close()
        res.append(sum(int((a != b).sum()) for a, b in zip(o, ref)))
    print(name, res, flush=True)
