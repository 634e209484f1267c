#!/usr/bin/env python
"""Record one fused launch's DRAM traffic (ncu --set full capture) in profiles/traffic.json.

    python tools/traffic_from_ncu.py REP.ncu-rep CONFIG LAYOUT N_SSTAR [note]

bench.py reads profiles/traffic.json[CONFIG][LAYOUT] for roofline.traffic (bytes per S* x
batch) and says it was not measured in the run itself."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(rep, cfg, layout, n_sstar, note=""):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    def get(name):
        i = hdr.index(name)
        v = float(vals[i].replace(",", ""))
        u = units[i].strip().lower()
        return v * {"gbyte": 1e9, "mbyte": 1e6, "kbyte": 1e3, "byte": 1.0}.get(u, 1.0)
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    kname = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "fused_kernel"
    n = int(n_sstar)
    p = os.path.join(ROOT, "profiles", "traffic.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    entry = d.setdefault(cfg, {})
    entry.setdefault("layouts", {})[layout] = {
        "dram_bytes_per_sstar": (rd + wr) / n, "read": rd, "write": wr, "sstar": n, "kernel": kname[:80],
        "source": f"ncu --set full, one full-size fused launch ({os.path.basename(rep)}) {note}".strip()}
    json.dump(d, open(p, "w"), indent=1)
    print(json.dumps(entry["layouts"][layout]))


if __name__ == "__main__":
    main(*sys.argv[1:])
