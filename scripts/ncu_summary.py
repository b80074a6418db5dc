"""Summarise ncu captures into profiles/ (run here, on the CPU box, after gpurun).

    python scripts/ncu_summary.py --tag r01 --rep vfa=gpurun_out/prof_vfa.ncu-rep \
        --rep fa=gpurun_out/prof_fa.ncu-rep --launches gpurun_out/launches.csv \
        [--flops 8.796e12] [--bench gpurun_out/bench.json]

Writes profiles/ncu_<tag>.md (human summary) and updates profiles/ncu_summary.json
(read by bench.py for roofline.traffic).
"""

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe % (MMA math)"),
    ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "tc pipe % (incl. TMEM traffic)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) inst %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "FMA-heavy pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe % (FMNMX, conversions)"),
    ("sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active", "TMEM inst %"),
    ("sm__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC per SM"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__cycles_active.avg", "SM active cycles"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
]
STALLS = ["long_scoreboard", "barrier", "wait", "no_instructions", "branch_resolving", "selected",
          "short_scoreboard", "math_pipe_throttle", "mio_throttle", "not_selected"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (vals[i], units[i]) for i, h in enumerate(hdr)}


def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return float(v.replace(",", "")) * scale


def to_seconds(v, u):
    scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
    return float(v.replace(",", "")) * scale.get(u, 1e-9)


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ci = {h: j for j, h in enumerate(hdr)}
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[ci["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ci["Kernel Name"]]
        name = name.split("(")[0][:70]
        agg[name][0] += 1
        agg[name][1] += float(r[ci["Metric Value"]].replace(",", ""))
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--rep", action="append", default=[], help="label=path.ncu-rep")
    ap.add_argument("--launches")
    ap.add_argument("--flops", type=float, default=8.796093022208e12)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    md = [f"# ncu summary {a.tag}", ""]
    if a.note:
        md += [a.note, ""]
    summary = {"tag": a.tag, "kernels": {}}
    for spec in a.rep:
        label, path = spec.split("=", 1)
        m = raw(path)
        md += [f"## {label}: `{os.path.basename(path)}`", "", "| metric | value |", "|---|---|"]
        rec = {}
        for key, desc in METRICS:
            if key in m:
                v, u = m[key]
                md.append(f"| {desc} (`{key}`) | {v} {u} |")
                rec[key] = [v, u]
        stall = {}
        for s in STALLS:
            key = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if key in m:
                stall[s] = float(m[key][0].replace(",", "") or 0)
        tot = sum(stall.values()) or 1
        md.append("| stall mix (pc sampling) | " + ", ".join(f"{k} {v / tot:.0%}" for k, v in
                                                              sorted(stall.items(), key=lambda kv: -kv[1])) + " |")
        if "dram__bytes_read.sum" in m:
            traffic = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
            rec["dram_bytes_per_launch"] = traffic
            md.append(f"| DRAM traffic per launch | {traffic / 1e6:.1f} MB |")
        if "gpu__time_duration.sum" in m:
            t = to_seconds(*m["gpu__time_duration.sum"])
            md.append(f"| algorithmic TFLOP/s at ncu duration (cold, serialised) | {a.flops / t / 1e12:.1f} |")
        summary["kernels"][label] = rec
        md.append("")
    if a.launches:
        agg = launches(a.launches)
        tot = sum(v[1] for v in agg.values())
        md += ["## launch list (ncu --metrics gpu__time_duration.sum, cold and serialised: compare shares)", "",
               "| launches | total ms | share | kernel |", "|---|---|---|---|"]
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            md.append(f"| {n} | {t / 1e6:.3f} | {t / tot:.1%} | `{k}` |")
        md.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"ncu_{a.tag}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    vfa = summary["kernels"].get("vfa")
    if vfa and "dram_bytes_per_launch" in vfa:
        js = {"tag": a.tag, "attention_kernel": {"label": "vfa", "dram_bytes_per_launch": vfa["dram_bytes_per_launch"]},
              "kernels": summary["kernels"]}
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w") as f:
            json.dump(js, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
