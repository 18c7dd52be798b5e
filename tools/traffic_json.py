"""Write profiles/ncu_traffic.json entries from an ncu dram csv of tools/prof_one.py
(2 steps: prologue, row, col, row, final).  Since the interior segments run in their
own launch (NOEND), one kernel KIND is several launches in a row;
the entry is their summed dram bytes, matching bench.py's per-kind launch time
(one CUDA-event bracket around all launches of the kind).

    python tools/traffic_json.py profiles/r01h/dram_cfd.csv cfd 16384 [suffix]
"""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODE_KIND = {"0": "sweep", "1": "final", "2": "prologue"}


def launches(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    iid, ik, im, iv = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    out = {}
    for r in rows[1:]:
        d = out.setdefault(int(r[iid]), {"name": r[ik]})
        d[r[im]] = float(r[iv].replace(",", ""))
    return [out[k] for k in sorted(out)]


def main():
    path, method, n = sys.argv[1], sys.argv[2], sys.argv[3]
    suffix = sys.argv[4] if len(sys.argv) > 4 else ""
    L = launches(path)
    # group consecutive launches of the same MODE into kinds; the sweep groups are
    # row, col, row (2 steps), then final
    groups = []
    for d in L:
        args = re.search(r"adi_line_kernel<([^>]*)>", d["name"]).group(1).split(", ")
        # template args: METHOD, M, NW, MODE, EDGE, HET, FULL, NOEND[, PACK]
        mode = args[3]
        pack = len(args) > 8 and args[8] == "1"
        noend = args[7] == "1" and not pack
        # a kind = its interior (NOEND) launch followed by its line-end / generic launches
        # (and, in the fragment plan, its PACK launch of the middle fragments)
        if groups and groups[-1][0] == mode and not noend:
            groups[-1][1].append(d)
        else:
            groups.append((mode, [d]))
    names = []
    sweeps = 0
    for mode, _ in groups:
        if MODE_KIND[mode] == "sweep":
            names.append(("row", "col")[sweeps % 2])
            sweeps += 1
        else:
            names.append(MODE_KIND[mode])
    tj = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    T = json.load(open(tj)) if os.path.exists(tj) else {}
    seen = set()
    for (mode, ds), kind in zip(groups, names):
        if kind not in ("row", "col") or kind in seen:
            continue
        seen.add(kind)
        byt = sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in ds)
        key = f"{method}_{kind}_{n}{suffix}"
        T[key] = {"dram_bytes_per_launch": byt,
                  "source": f"{os.path.relpath(path, ROOT)} (ncu dram__bytes_read/write.sum, {n}^2, "
                            f"{len(ds)} launches of the kind summed: "
                            + ", ".join(d["name"].split("(")[0] for d in ds) + ")"}
        print(key, byt)
    json.dump(T, open(tj, "w"), indent=1)


if __name__ == "__main__":
    main()
