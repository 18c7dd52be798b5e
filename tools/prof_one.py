"""Minimal driver for ncu: one ADI call of `steps` steps on an n x n MMS grid
(argv[4] == "media": in the bench's heterogeneous medium, NEXT row f3; argv[1] ==
"shots": the config-5 batch of 8 Ricker shots of 4096^2, MFD)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_07583_b200 as adi
from adi_inputs import CFD, MFD
from bench import make_problem

if sys.argv[1] == "shots":
    # config 5: a batch of 8 Ricker shots of 4096^2 nodes (bench.py --shots), MFD
    import numpy as np
    from bench import SHOT_N, shot_problems
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    probs = shot_problems(0, 8, steps + 2, 8)
    p0 = probs[0]
    s = adi.AdiSolver(SHOT_N, SHOT_N, p0.h, p0.dt, 1.0, MFD, batch=8)
    for kv in filter(None, os.environ.get("ADI_SET", "").split(",")):   # knobs, e.g. ADI_FRAG_TILES=0
        k, v = kv.split("=")
        s.set_param(getattr(adi, k), float(v))
    s.set_point_sources([p.src[0] for p in probs], [p.src[1] for p in probs], p0.gf)
    s.set_fields(*(np.zeros((8,) + a.shape) for a in (p0.U, p0.V, p0.W)))
    s.step(steps)
    s.get_fields()
    print("ok shots", SHOT_N, steps)
    sys.exit(0)
method = {"cfd": CFD, "mfd": MFD, "cfd_full": 2}[sys.argv[1]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
media = len(sys.argv) > 4 and sys.argv[4] == "media"
p = make_problem(method, n, steps + 2, 8, media)
s = adi.AdiSolver.from_problem(p)
if method == 2:
    from bench import ABSORB_NB, ABSORB_A
    s.set_param(adi.ADI_ABSORB_WIDTH, ABSORB_NB)
    s.set_param(adi.ADI_ABSORB_RATE, ABSORB_A)
s.step(steps)
s.get_fields()
print("ok", sys.argv[1], n, steps, "media" if media else "")
