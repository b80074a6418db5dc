"""Aggregate warp-stall samples of an `ncu --page source --print-source=cuda,sass --csv` export by CUDA source line."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file, cur_line, src = None, None, {}
agg = defaultdict(lambda: [0, defaultdict(int)])
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if len(r) > 4 and r[0].isdigit():
        cur_line = (cur_file, int(r[0]))
        src[cur_line] = r[1].strip()[:80]
        continue
    if len(r) > 4 and r[2].startswith("0x") and hdr:
        s = int(r[4] or 0)
        a = agg[cur_line]
        a[0] += s
        for h, i in hdr.items():
            if h.startswith("stall_") and "Not Issued" not in h and r[i]:
                a[1][h[6:]] += int(r[i])
tot = sum(v[0] for v in agg.values())
print("total", tot)
for k, (s, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    mix = ",".join(f"{a}:{b}" for a, b in sorted(st.items(), key=lambda kv: -kv[1])[:3])
    print(f"{s:8d} {s/tot:6.2%} {k[0]}:{k[1]:<5d} {src.get(k,'')[:60]:60s} {mix}")
