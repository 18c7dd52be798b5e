import sys; sys.path.insert(0, '.')
import numpy as np, oracle, paper_2006_07583_b200 as adi
from adi_inputs import CFD, random_problem
for n, steps in ((1601, 1), (1001, 1)):
    p = random_problem(CFD, n, seed=5, steps=steps)
    s = adi.AdiSolver.from_problem(p)
    if n == 1001: s.set_param(adi.ADI_TILE_CHUNKS, 20)
    s.step(steps); g = s.get_fields()
    o = oracle.run(p.method, p.nx, p.ny, p.h, p.dt, p.c, p.K, p.U, p.V, p.W, nsteps=steps, **p.oracle_kwargs())
    for name, a, b in zip("UVW", g, o):
        d = np.abs(a - b); scale = np.abs(b).max()
        bad = np.argwhere(d > 1e-9 * scale)
        print(n, name, a.shape, 'maxrel', d.max() / scale, 'nbad', len(bad))
        if len(bad):
            ys, xs = bad[:, 0], bad[:, 1]
            print('   rows', np.unique(ys)[:12], '... cols', np.unique(xs)[:12], '...', np.unique(xs)[-6:])
