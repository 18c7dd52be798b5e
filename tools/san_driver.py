"""Driver for compute-sanitizer (tools/sanitize.sh): every kernel kind of libadi.so on
small grids -- prologue, ADI-rows, ADI-columns (fused a2), FINAL, the carry kernel, the
heterogeneous-media (HET) and full-matrix (FULL) instantiations, the stopping-rule
attempts and decision kernel, the thread-per-line kernels, a band-local group with the
loopback halo exchange, and a graph-captured call.  Usage: python tools/san_driver.py N"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2006_07583_b200 as adi
from adi_inputs import CFD, MFD, random_problem

n = int(sys.argv[1]) if len(sys.argv) > 1 else 41
for method in (CFD, MFD):
    # plain: prologue, rows, cols, carry kernel, then FINAL (carry off), thread kernels
    for thread in (0, 1):
        if thread and n > 250:
            continue
        p = random_problem(method, n, seed=1, steps=8)
        s = adi.AdiSolver.from_problem(p)
        s.set_param(adi.ADI_THREAD_LINES, thread)
        s.step(2)
        s.step(1)                      # after a carry (no prologue)
        s.set_param(adi.ADI_CARRY, 0)
        s.step(1)                      # FINAL
        s.set_param(adi.ADI_GRAPH, 1)
        s.step(2)                      # captured
        s.get_fields()
        s.close()
    # media (HET kernels)
    p = random_problem(method, n, seed=2, steps=2, media=True)
    s = adi.AdiSolver.from_problem(p)
    s.step(2)
    s.get_fields()
    s.close()
    # stopping rule (KM_*_T attempts + decide_sweeps_kernel)
    p = random_problem(method, n, seed=3, steps=2)
    p.K = 10
    s = adi.AdiSolver.from_problem(p)
    s.set_param(adi.ADI_EPS, 1e-6)
    s.set_param(adi.ADI_K_MIN, 3)
    s.step(2)
    s.get_fields()
    s.close()
    # band-local ranks with the loopback exchange (overlapped column sweep)
    if n >= 120:
        hs = adi.adi_create_dist_local(p.nx, p.ny, p.h, p.dt, p.c, method, 1, 2)
        ss = [adi.AdiSolver.adopt(h, p.nx, p.ny, p.h, p.dt, p.c, method) for h in hs]
        for x in ss:
            x.set_fields(p.U, p.V, p.W)
            x.set_source(p.phi, None, p.gf)
        adi.adi_step_dist_local(hs, 1)
        adi.adi_step_dist_local(hs, 1)
        for x in ss:
            x.close()
# full-matrix variant with a Cerjan layer (FULL kernels)
rng = np.random.default_rng(0)
h = 1.0 / (n - 1)
s = adi.AdiSolver(n, n, h, 0.91 * h, 1.0, adi.ADI_CFD_FULL)
s.set_fields(*(rng.standard_normal((n, n)) for _ in range(3)))
s.set_source(rng.standard_normal((n, n)), None, rng.standard_normal(9))
s.set_param(adi.ADI_ABSORB_WIDTH, min(6, n // 4))
s.step(2)
s.get_fields()
s.close()
print("san_driver ok", n)
