"""the paper's accuracy study (Tables 3-4)
rerun on the GPU through the C-ABI.

For each method (CFD cfl 0.91, MFD cfl 0.81), each case Γ ∈ {0, Γ=k=2, Γ=k=9}
and N ∈ {16, 24, ..., 1024} cells: the Γ/k manufactured solution (eq. 11)
advanced to T_sim = 5T with K = 8, the unnormalised Frobenius error of the
interior pressure [G17] (and the rates in the h-weighted L2 norm, h times that
norm: rate + 1), the rates from consecutive N and the trimmed
average, next to the printed values of Tables 3-4
(tests/golden/paper_table{3,4}_*.txt).

Usage: [ADI_K=8] [ADI_ONLY=mfd|cfd] python tools/rate_study.py [out.json]
"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2006_07583_b200 as adi
from adi_inputs import CFD, MFD, MMS, mms_problem
from adi_inputs.mms import interior_error
from adi_inputs.rates import estimate_rates, trimmed_average

NS = [16, 24, 32, 48, 64, 96, 128, 256, 512, 1024]
CASES = {"gamma0": MMS(), "gamma2": MMS(gamma=2.0, k=2), "gamma9": MMS(gamma=9.0, k=9)}
T = 1.0 / math.sqrt(2.0)


def golden(name):
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
    rows = [l.split() for l in open(os.path.join(root, name)) if l.strip() and not l.startswith("#")]
    return {r[0]: [float(x) for x in r[1:]] for r in rows}


KSW = int(os.environ.get("ADI_K", "8"))
ONLY = os.environ.get("ADI_ONLY", "")   # e.g. "mfd" to run one method


def run(method, case, N):
    p = mms_problem(method, N + 1, case, t_sim=5 * T)
    s = adi.AdiSolver.from_problem(p)
    if KSW != 8:
        s.set_param(adi.ADI_K_SWEEPS, KSW)
    t0 = time.perf_counter()
    s.step(p.meta["steps"])
    U, _, _ = s.get_fields()
    dt = time.perf_counter() - t0
    s.close()
    return interior_error(p, U, p.meta["t_end"]), p.meta["steps"], dt


def main(out):
    res = {}
    for method, table in ((MFD, "paper_table4_mfd_rates.txt"), (CFD, "paper_table3_cfd_rates.txt")):
        mname = ("cfd", "mfd")[method]
        if ONLY and mname != ONLY:
            continue
        paper = golden(table)
        res[mname] = {}
        for ci, (cname, case) in enumerate(CASES.items()):
            errs, steps, secs = [], [], []
            for N in NS:
                e, st, dt = run(method, case, N)
                errs.append(e)
                steps.append(st)
                secs.append(dt)
            rates = estimate_rates(errs, NS)
            # the h-weighted L2 norm is h * (unnormalised Frobenius norm): rate + 1
            rates_h = [r + 1.0 for r in rates]
            printed = [paper[str(N)][ci] for N in NS[1:] if str(N) in paper]
            res[mname][cname] = {
                "N": NS, "steps": steps, "error": errs, "rates": rates,
                "trimmed_average": trimmed_average(rates),
                "rates_h_weighted_L2": rates_h, "trimmed_average_h_weighted_L2": trimmed_average(rates_h),
                "paper_rates": printed, "paper_trimmed_average": paper["AVG"][ci],
                "gpu_seconds": secs}
            print(f"{mname} {cname}: trimmed avg {trimmed_average(rates):.2f} "
                  f"(h-weighted L2 {trimmed_average(rates_h):.2f}; paper {paper['AVG'][ci]:.2f}); rates "
                  + " ".join(f"{r:.2f}" for r in rates), flush=True)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "rate_study.json")
