"""Same-box A/B of BUILD variants of libadi.so (compile-time knobs): run as
    python tools/ab_lib.py A.so,B.so,... [n] [steps] [rounds]
Each variant runs in its own child process (a library is loaded once per process),
interleaved over `rounds`, on the bench workload (16384^2 MMS, K = 8, dense
source); prints ms/step and per-kind kernel times, and checks that every variant
returns the same fields bit for bit (a knob must not change results)."""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, json, hashlib
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2006_07583_b200 as adi
adi.LIB_PATH = LIBP
from adi_inputs import CFD, MFD
from bench import make_problem
out = {}
stream = torch.cuda.current_stream()
for m, name in ((MFD, "mfd"), (CFD, "cfd")):
    p = make_problem(m, N, 2 * STEPS + 8, 8)
    s = adi.AdiSolver.from_problem(p, stream=stream.cuda_stream)
    s.step(2)
    U = s.get_fields()[0]
    h = hashlib.sha1(np.ascontiguousarray(U).tobytes()).hexdigest()[:12]
    s.step(1)
    torch.cuda.synchronize()
    s.set_param(adi.ADI_TIMING, 1); s.kernel_times()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream); s.step(STEPS); e1.record(stream); e1.synchronize()
    kt = {k: v[0] / v[1] for k, v in s.kernel_times().items() if v[1]}
    s.close()
    out[name] = {"ms": e0.elapsed_time(e1) / STEPS, "k": kt, "hash": h}
print("RESULT " + json.dumps(out))
"""


def main():
    libs = sys.argv[1].split(",")
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    res = {l: [] for l in libs}
    for r in range(rounds):
        for l in libs:
            code = CHILD.replace("ROOT", repr(ROOT)).replace("LIBP", repr(os.path.abspath(l))) \
                .replace("STEPS", str(steps)).replace("N,", f"{n},")
            o = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT)
            line = [x for x in o.stdout.splitlines() if x.startswith("RESULT ")]
            if not line:
                print(l, "FAILED", o.stderr[-800:])
                continue
            res[l].append(json.loads(line[0][7:]))
    for l in libs:
        for m in ("mfd", "cfd"):
            xs = [d[m] for d in res[l]]
            if not xs:
                continue
            best = min(xs, key=lambda d: d["ms"])
            print(f"{os.path.basename(l):14s} {m}: ms/step " + " ".join(f"{d['ms']:.3f}" for d in xs)
                  + " | best kernels " + " ".join(f"{k} {v:.3f}" for k, v in best["k"].items())
                  + f" | U hash {sorted(set(d['hash'] for d in xs))}")
    sys.stdout.flush()


if __name__ == "__main__":
    main()
