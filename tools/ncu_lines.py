"""Aggregate warp-stall samples (with the top stall reasons) and executed
instructions per CUDA source line (ncu --page source --print-source cuda,sass).
Usage: ncu_lines.py rep [kernel#] [top]"""
import csv, io, subprocess, sys

def main(rep, kidx=0, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    parts = out.split('"File Path"')[1:]
    # one block per (kernel, file); pick the blocks of kernel kidx (function name row)
    funcs = []
    for p in parts:
        rows = list(csv.reader(io.StringIO('"File Path"' + p)))
        funcs.append((rows[1][1], rows))
    names = []
    for f, _ in funcs:
        if f not in names:
            names.append(f)
    fname = names[kidx]
    lines = []
    reasons_tot = {}
    for f, rows in funcs:
        if f != fname:
            continue
        fpath = rows[0][1].split("/")[-1]
        hdr = rows[2]
        iW = hdr.index("Warp Stall Sampling (All Samples)")
        iE = hdr.index("Instructions Executed")
        rcols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        for r in rows[3:]:
            if len(r) < len(hdr) or not r[0]:
                continue
            try:
                ln = int(r[0])
                w = float(r[iW]) if r[iW] not in ("-", "") else 0.0
                e = float(r[iE]) if r[iE] not in ("-", "") else 0.0
            except ValueError:
                continue
            rs = {}
            for i, h in rcols:
                try:
                    v = float(r[i])
                except ValueError:
                    v = 0.0
                rs[h[6:]] = v
                reasons_tot[h[6:]] = reasons_tot.get(h[6:], 0) + v
            lines.append((fpath, ln, r[1], w, e, rs))
    tw = sum(x[3] for x in lines) or 1
    te = sum(x[4] for x in lines) or 1
    print(fname[:110], f"| samples {tw:.0f} warp-instr {te:.3e}")
    rt = sum(reasons_tot.values()) or 1
    print("reasons:", ", ".join(f"{k}={100*v/rt:.1f}%" for k, v in sorted(reasons_tot.items(), key=lambda x: -x[1])[:9]))
    for fp, ln, src, w, e, rs in sorted(lines, key=lambda x: -x[3])[:top]:
        s = sum(rs.values()) or 1
        rtxt = " ".join(f"{k}:{100*v/s:.0f}" for k, v in sorted(rs.items(), key=lambda x: -x[1])[:3] if v > 0)
        print(f"{fp[:14]:14s}{ln:>5} stall {100*w/tw:5.1f}%  inst {100*e/te:5.1f}%  [{rtxt}]  {src.strip()[:70]}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0, int(sys.argv[3]) if len(sys.argv) > 3 else 30)
