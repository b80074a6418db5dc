"""Per setmaxnreg region: instruction count, spills (STL/LDL), FFMA2/FADD2/MUFU/LDTM/STTM/UTCHMMA counts."""
import re
import sys
from collections import Counter

txt = open(sys.argv[1]).read()
pat = sys.argv[2] if len(sys.argv) > 2 else "Li128ELi128ELi2ELi1E"
for f in re.split(r"\n\s*Function : ", txt)[1:]:
    name = f.split("\n")[0]
    if pat not in name:
        continue
    print("==", name[:90])
    region = "pre"
    cnt = {}
    for ln in f.split("\n"):
        m = re.search(r"USETMAXREG\.(\S+)\s*(?:\S+,\s*)?(0x[0-9a-f]+)", ln)
        if m:
            region = m.group(1)[:5] + m.group(2) + "@" + re.search(r"/\*([0-9a-f]+)\*/", ln).group(1)
        m = re.search(r"/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", ln)
        if not m:
            continue
        op = m.group(2)
        c = cnt.setdefault(region, Counter())
        c["total"] += 1
        for key in ("STL", "LDL", "FFMA2", "FADD2", "FMUL2", "MUFU.EX2", "LDTM", "STTM", "UTCHMMA", "UTCBAR",
                    "F2FP", "FMNMX", "FFMA", "FADD", "IMAD", "SHF", "LEA", "BRA", "SYNCS"):
            if op == key or op.startswith(key + "."):
                c[key] += 1
    for reg, c in cnt.items():
        print(f"  {reg:28s}", dict(c))
