import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2006_07583_b200 as adi
from adi_inputs import CFD, MFD, random_problem
for method, n in ((MFD, 77), (CFD, 77)):
    for steps in (1, 3):
        p = random_problem(method, n, seed=11, steps=steps)
        s = adi.AdiSolver.from_problem(p); s.step(steps); ref = s.get_fields(); s.close()
        for r in range(10):
            st = torch.cuda.Stream()
            s = adi.AdiSolver.from_problem(p, stream=st.cuda_stream); s.step(steps); o = s.get_fields(); s.close()
            for name, a, b in zip("UVW", o, ref):
                d = np.argwhere(a != b)
                if len(d):
                    print(("CFD", "MFD")[method], "steps", steps, "run", r, name, a.shape, "n diff", len(d),
                          "rows", sorted(set(d[:, 0].tolist()))[:10], "cols", sorted(set(d[:, 1].tolist()))[:10], flush=True)
