"""Executed-instruction mix by SASS opcode (ncu --page source --print-source sass)."""
import csv, io, subprocess, sys, collections

def main(rep, kidx=0, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    parts = out.split('"Address"')
    # each kernel block starts with a header row containing "Address"
    blocks = ['"Address"' + p for p in parts[1:]]
    rows = list(csv.reader(io.StringIO(blocks[kidx])))
    hdr = rows[0]
    iS = hdr.index("Source"); iE = hdr.index("Instructions Executed")
    iW = hdr.index("Warp Stall Sampling (All Samples)")
    mix = collections.Counter(); st = collections.Counter()
    for r in rows[1:]:
        if len(r) < len(hdr):
            continue
        try:
            e = float(r[iE] or 0); w = float(r[iW] or 0)
        except ValueError:
            continue
        toks = r[iS].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        mix[op] += e; st[op] += w
    te = sum(mix.values()) or 1; tw = sum(st.values()) or 1
    print(f"warp-instr {te:.3e}")
    for op, e in mix.most_common(top):
        print(f"{op:10s} inst {100*e/te:5.1f}%  stall {100*st[op]/tw:5.1f}%")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0, int(sys.argv[3]) if len(sys.argv) > 3 else 25)
