import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2006_07583_b200 as adi
from adi_inputs import CFD, MFD, random_problem
p = random_problem(MFD, 77, seed=11, steps=3)
def run(stream=None, asy=False, reps=1):
    outs = []
    for _ in range(reps):
        st = torch.cuda.Stream() if stream == "new" else None
        s = adi.AdiSolver.from_problem(p, **({"stream": st.cuda_stream} if st else {}))
        if asy:
            pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
            hU, hV, hW = pin(p.U), pin(p.V), pin(p.W)
            o = [torch.empty(x.shape, dtype=torch.float64).pin_memory().numpy() for x in (hU, hV, hW)]
            adi.adi_set_fields_async(s.handle, hU, hV, hW); s.step(3); adi.adi_get_fields_async(s.handle, *o)
            (st.synchronize() if st else torch.cuda.synchronize())
        else:
            s.step(3); o = s.get_fields()
        s.close(); outs.append(o)
    return outs
ref = run()[0]
for label, kw in (("default+sync x3", dict(reps=3)), ("new+sync", dict(stream="new", reps=3)),
                  ("default+async", dict(asy=True, reps=3)), ("new+async", dict(stream="new", asy=True, reps=3))):
    outs = run(**kw)
    print(label, [[float(np.abs(a - b).max()) for a, b in zip(o, ref)] for o in outs])
