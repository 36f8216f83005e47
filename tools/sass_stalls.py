"""Developer tool: per-region / per-instruction stall samples from an ncu source-page CSV
(ncu -i X.ncu-rep --page source --csv --print-source sass).
usage: sass_stalls.py FILE [lo_hex hi_hex]   (offsets relative to the kernel start)"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
base = int(data[0][ix["Address"]], 16)
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 40
agg = collections.Counter()
for r in data:
    a = int(r[ix["Address"]], 16) - base
    if not lo <= a < hi:
        continue
    src = r[ix["Source"]].strip()
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    n = int(r[ix["Instructions Executed"]] or 0)
    st = {c[6:]: int(r[ix[c]]) for c in cols if r[ix[c]] not in ("", "0")}
    for k, v in st.items():
        agg[k] += v
    if len(sys.argv) > 2 and (s or "SYNCS" in src or "BAR" in src):
        print(f"{a:6x} {src[:60]:60s} {s:5d} {n:8d} {st}")
print(agg.most_common())
