"""Summarise an .ncu-rep: key metrics, stall breakdown, top-stall SASS lines."""
import csv, subprocess, sys, io
from collections import Counter

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sectors_srcunit_tex.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]

def main(rep, nsass=15):
    hdr, units, rows = raw(rep)
    for r in rows:
        d = dict(zip(hdr, r))
        print("=====", d["Kernel Name"][:90])
        for k in KEYS:
            if k in d:
                print(f"   {k:70s} {d[k]} {units[hdr.index(k)]}")
        st = {h: float(v) for h, v in d.items() if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued") and v not in ("", "n/a")}
        tot = sum(st.values()) or 1
        print("   stalls:", ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_','')}={100*v/tot:.1f}%" for h, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
    secs = []; cur = None
    for l in out.split("\n"):
        if l.startswith('"Kernel Name"'):
            cur = [l]; secs.append(cur)
        elif cur is not None:
            cur.append(l)
    for sec in secs:
        rr = list(csv.reader(sec[1:]))
        h = rr[0]; data = [r for r in rr[1:] if len(r) == len(h)]
        iS, iW = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
        tot = sum(float(r[iW] or 0) for r in data) or 1
        c = Counter()
        for r in data:
            toks = r[iS].split()
            op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "")
            c[op.split(".")[0]] += float(r[iW] or 0)
        print("---", sec[0][:100])
        print("   by opcode:", ", ".join(f"{k}={100*v/tot:.1f}%" for k, v in c.most_common(10)))
        for r in sorted(data, key=lambda r: -float(r[iW] or 0))[:nsass]:
            print(f"   {100*float(r[iW] or 0)/tot:5.1f}%  {r[iS][:90]}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 15)
