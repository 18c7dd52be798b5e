"""Cost of the inner stopping rule (ADI_EPS > 0) at the benchmark size: device time
per step with fixed K = 8 vs the rule with k_max = 8, k_min = 6, eps chosen so that
stages stop at 6-7 sweeps; the sweeps chosen are reported."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2006_07583_b200 as adi
from adi_inputs import CFD, MFD, MMS, mms_problem

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
steps = 6
for method in (MFD, CFD):
    p = mms_problem(method, n, MMS(), steps=40)
    s = adi.AdiSolver.from_problem(p, stream=torch.cuda.current_stream().cuda_stream)
    res = {}
    for eps in (0.0, 1e-6, 1e-3, 1.0):
        s.set_param(adi.ADI_EPS, eps)
        s.set_param(adi.ADI_K_MIN, 6)
        s.set_fields(p.U, p.V, p.W)
        s.step(2)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.step(steps)
        e1.record()
        e1.synchronize()
        res[eps] = (e0.elapsed_time(e1) / steps, adi.adi_get_last_sweeps(s.handle))
        s.m = 0
    print(("CFD", "MFD")[method], {k: (round(v[0], 3), v[1]) for k, v in res.items()}, flush=True)
