"""Summarise an `ncu --page source --print-source=sass --csv` export: hottest SASS lines and stall mix."""
import csv
import sys
from collections import Counter

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
hdr = rows[1]
data = rows[2:]
ci = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
items = []
for r in data:
    try:
        s = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    st = {h: int(r[ci[h]] or 0) for h in stall_cols}
    tot.update(st)
    items.append((s, r[ci["Address"]], r[ci["Source"]], st))
allsum = sum(x[0] for x in items)
print("total samples", allsum)
print("stall mix:", ", ".join(f"{k[6:]}={v/allsum:.1%}" for k, v in tot.most_common(10)))
for s, a, src, st in sorted(items, key=lambda x: -x[0])[:top]:
    mix = ",".join(f"{k[6:]}:{v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3] if v)
    print(f"{s:7d} {s/allsum:6.2%} {a:>6s} {src[:70]:70s} {mix}")
