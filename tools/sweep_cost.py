"""Per-sweep vs fixed cost of the line kernels: time the row/col kernels at several K."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2006_07583_b200 as adi
from adi_inputs import CFD, MFD, MMS, mms_problem

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
for method in (MFD, CFD):
    p = mms_problem(method, n, MMS(), steps=40)
    s = adi.AdiSolver.from_problem(p, stream=torch.cuda.current_stream().cuda_stream)
    res = {}
    for K in (1, 4, 8, 16, 32):
        s.set_param(adi.ADI_K_SWEEPS, K)
        s.set_fields(p.U, p.V, p.W)
        s.step(2)
        s.set_param(adi.ADI_TIMING, 1)
        s.kernel_times()
        s.step(3)
        kt = s.kernel_times()
        s.set_param(adi.ADI_TIMING, 0)
        res[K] = kt["row"][0] / kt["row"][1]
        s.m = 0
    Ks = np.array(sorted(res)); ts = np.array([res[k] for k in Ks])
    b, a = np.polyfit(Ks, ts, 1)
    pts = n * n
    dp_per_sweep = {MFD: 8, CFD: 12}[method] * pts / (148 * 64 * 1.965e9) * 1e3
    print(("CFD", "MFD")[method], "row kernel ms by K:", {int(k): round(v, 3) for k, v in res.items()},
          f"fixed {a:.3f} ms, per sweep {b:.3f} ms (DP bound {dp_per_sweep:.3f} ms -> {dp_per_sweep/b:.0%})")
