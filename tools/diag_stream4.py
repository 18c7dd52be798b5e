import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2006_07583_b200 as adi
from adi_inputs import CFD, MFD, random_problem
p = random_problem(MFD, 77, seed=11, steps=1)
s = adi.AdiSolver.from_problem(p); s.step(1); ref = s.get_fields(); s.close()
def trial(sync_after_setup, sync_after_step):
    st = torch.cuda.Stream()
    s = adi.AdiSolver.from_problem(p, stream=st.cuda_stream)
    if sync_after_setup: torch.cuda.synchronize()
    s.step(1)
    if sync_after_step: torch.cuda.synchronize()
    o = s.get_fields(); s.close()
    return sum(int((a != b).sum()) for a, b in zip(o, ref))
for a_, b_ in ((False, False), (True, False), (False, True), (True, True)):
    print("sync setup", a_, "sync step", b_, [trial(a_, b_) for _ in range(8)], flush=True)
