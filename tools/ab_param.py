"""Same-box A/B of a performance knob (adi_set_param): for each method, one handle on
the bench workload (16384^2 MMS, K = 8, dense source); the values are interleaved
over several rounds so clock drift hits them alike.  Prints ms/step per value and
the per-kind kernel times.  The knob must not change results: the fields after the
runs are compared bit for bit between the values.

    python tools/ab_param.py KEY v1,v2,... [n] [steps] [rounds] [methods]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2006_07583_b200 as adi  # noqa: E402
from adi_inputs import CFD, MFD  # noqa: E402
from bench import make_problem  # noqa: E402

key = int(sys.argv[1])
vals = [float(v) for v in sys.argv[2].split(",")]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 3
methods = [{"mfd": MFD, "cfd": CFD}[m] for m in (sys.argv[6] if len(sys.argv) > 6 else "mfd,cfd").split(",")]
stream = torch.cuda.current_stream()
for m in methods:
    p = make_problem(m, n, (rounds * len(vals) + 1) * (steps + 2) + 4, 8)
    times = {v: [] for v in vals}
    kts = {v: {} for v in vals}
    res = {}
    for v in vals:
        # identical start per value for the bitwise comparison
        s = adi.AdiSolver.from_problem(p, stream=stream.cuda_stream)
        s.set_param(key, v)
        s.step(2)
        res[v] = s.get_fields()[0][:: max(n // 512, 1), :: max(n // 512, 1)].copy()
        s.close()
    base = res[vals[0]]
    same = {v: bool(np.array_equal(res[v], base)) for v in vals}
    s = adi.AdiSolver.from_problem(p, stream=stream.cuda_stream)
    s.step(2)
    for r in range(rounds):
        for v in vals:
            s.set_param(key, v)
            s.step(1)
            torch.cuda.synchronize()
            s.set_param(adi.ADI_TIMING, 1)
            s.kernel_times()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            s.step(steps)
            e1.record(stream)
            e1.synchronize()
            times[v].append(e0.elapsed_time(e1) / steps)
            for k, (ms, cnt) in s.kernel_times().items():
                if cnt:
                    kts[v].setdefault(k, []).append(ms / cnt)
            s.set_param(adi.ADI_TIMING, 0)
    s.close()
    name = {MFD: "mfd", CFD: "cfd"}[m]
    for v in vals:
        t = times[v]
        print(f"{name} key={key} value={v:g}: ms/step min {min(t):.3f} med {sorted(t)[len(t) // 2]:.3f} "
              f"| kernels " + " ".join(f"{k} {min(x):.3f}" for k, x in kts[v].items())
              + f" | bitwise-equal to value {vals[0]:g}: {same[v]}")
    sys.stdout.flush()
