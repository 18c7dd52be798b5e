"""Aggregate warp-stall samples and executed instructions per CUDA source line
(ncu --page source --print-source cuda,sass).  Usage: ncu_lines.py rep [kernel#] [top]"""
import csv, io, subprocess, sys

def main(rep, kidx=0, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    parts = out.split('"File Path"')[1:]
    blk = parts[kidx]
    rows = list(csv.reader(io.StringIO(blk)))
    # rows[0] = file path row remainder, rows[1] = function name, rows[2] = header
    hdr = rows[2]
    iW = hdr.index("Warp Stall Sampling (All Samples)")
    iE = hdr.index("Instructions Executed")
    lines = []
    for r in rows[3:]:
        if len(r) < len(hdr) or not r[0]:
            continue
        try:
            w = float(r[iW]) if r[iW] not in ("-", "") else 0.0
            e = float(r[iE]) if r[iE] not in ("-", "") else 0.0
            int(r[0])
        except ValueError:
            continue
        lines.append((int(r[0]), r[1], w, e))
    tw = sum(x[2] for x in lines) or 1
    te = sum(x[3] for x in lines) or 1
    print(rows[1][1][:110], f"| samples {tw:.0f} warp-instr {te:.3e}")
    for ln, src, w, e in sorted(lines, key=lambda x: -x[2])[:top]:
        print(f"{ln:>5} stall {100*w/tw:5.1f}%  inst {100*e/te:5.1f}%  {src.strip()[:90]}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0, int(sys.argv[3]) if len(sys.argv) > 3 else 30)
