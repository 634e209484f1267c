"""Summarise an ncu --page source --csv --print-source sass export: per-address-bucket stall
samples split by reason, plus the hottest instructions.  Usage: stall_regions.py file.csv [bucket_hex]"""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
bucket = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0x800
h = rows[1]
data = rows[2:]
ia = h.index("Address")
isrc = h.index("Source")
iex = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in reasons}
seen = set()
recs = []
for r in data:
    if r[ia] in seen:
        continue
    seen.add(r[ia])
    try:
        a = int(r[ia], 16)
    except ValueError:
        continue
    st = {c: int(r[idx[c]] or 0) for c in reasons}
    recs.append((a, r[isrc], int(r[iex] or 0), st))
recs.sort()
base = recs[0][0]
tot = sum(sum(st.values()) for *_, st in recs)
totr = collections.Counter()
for *_, st in recs:
    totr.update(st)
print("total samples", tot)
print("  ".join(f"{k[6:]}={100 * v / tot:.1f}%" for k, v in totr.most_common(8)))
b = collections.OrderedDict()
for a, src, ex, st in recs:
    k = (a - base) // bucket
    b.setdefault(k, collections.Counter()).update(st)
for k, c in b.items():
    s = sum(c.values())
    if s > 0.01 * tot:
        print(f"{k * bucket:6x} {100 * s / tot:5.1f}%  " + " ".join(f"{r[6:]}={v}" for r, v in c.most_common(4)))
print("hottest:")
for a, src, ex, st in sorted(recs, key=lambda x: -sum(x[3].values()))[:25]:
    s = sum(st.values())
    top = max(st, key=st.get)
    print(f"{a - base:6x} {100 * s / tot:5.1f}% ex={ex:8d} {top[6:]:10s} {src[:70]}")
