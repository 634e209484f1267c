#!/usr/bin/env python
"""Per-source-line instruction and stall-sample shares of one kernel in an ncu report.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = rows[2]
    ie = hdr.index("Instructions Executed")
    sm = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    res = []
    for r in rows[3:]:
        if r[0] == "":
            continue
        try:
            res.append((int(r[0]), r[1].strip(), int(r[ie]), int(r[sm]),
                        {hdr[i][6:]: int(r[i]) for i in stall_cols if r[i].isdigit() and int(r[i]) > 0}))
        except ValueError:
            pass
    tot = sum(x[2] for x in res) or 1
    tots = sum(x[3] for x in res) or 1
    agg = {}
    for x in res:
        for k, v in x[4].items():
            agg[k] = agg.get(k, 0) + v
    print(f"instructions {tot}  stall samples {tots}")
    print("stall mix: " + "  ".join(f"{k}={v / tots * 100:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
    res.sort(key=lambda x: -x[3])
    for ln, src, n, s, st in res[:top]:
        t3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        print(f"{ln:5d} inst {n / tot * 100:5.1f}%  stall {s / tots * 100:5.1f}%  {src[:64]:64s} {t3}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
