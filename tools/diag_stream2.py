import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2006_07583_b200 as adi
from adi_inputs import CFD, MFD, random_problem
for method, n in ((MFD, 77), (CFD, 77), (MFD, 1601), (CFD, 1601)):
    p = random_problem(method, n, seed=11, steps=3)
    s = adi.AdiSolver.from_problem(p); s.step(3); ref = s.get_fields(); s.close()
    bad = 0; reps = 12 if n < 1000 else 4
    for r in range(reps):
        st = torch.cuda.Stream()
        s = adi.AdiSolver.from_problem(p, stream=st.cuda_stream); s.step(3); o = s.get_fields(); s.close()
        if any(not np.array_equal(a, b) for a, b in zip(o, ref)): bad += 1
    print(("CFD", "MFD")[method], n, f"mismatches {bad}/{reps}", flush=True)
