import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2006_07583_b200 as adi
from adi_inputs import CFD, MFD, random_problem
p = random_problem(MFD, 77, seed=11, steps=1)
s = adi.AdiSolver.from_problem(p); s.step(1); ref = s.get_fields(); s.close()
res = []
for _ in range(16):
    s = adi.AdiSolver.from_problem(p); s.step(1); o = s.get_fields(); s.close()
    res.append(sum(int((a != b).sum()) for a, b in zip(o, ref)))
print("default stream", res)
cur = torch.cuda.current_stream()
res = []
for _ in range(16):
    s = adi.AdiSolver.from_problem(p, stream=cur.cuda_stream); s.step(1); o = s.get_fields(); s.close()
    res.append(sum(int((a != b).sum()) for a, b in zip(o, ref)))
print("torch current stream", cur.cuda_stream, res)
