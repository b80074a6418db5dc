"""A/B timing of library builds (tuning experiments; not bench values).

    python scripts/ab.py [--variant vfa] [--steps 20] NAME=path/to/lib.so[@SPLIT] [NAME=...]
Loads every build into one process and times them interleaved step by step on the C2 problem
(same inputs, same clock / power state), so small differences are attributable to the code.
Also checks every build's output is bitwise identical to the first one's where expected.
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, ClockSampler, Runner, causal_flops, make_inputs, time_interleaved  # noqa: E402
from paper_2604_12798_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--variant", default="vfa")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--k-block", type=int, default=128)
ap.add_argument("--head-dim", type=int, default=128)
ap.add_argument("--pair", action="store_true", help="also time every build with cta_pair=2")
ap.add_argument("--split", type=int, default=0, help="softmax_split for every runner (0: per-variant default)")
a = ap.parse_args()
cfg = dict(CONFIGS["c2"], d=a.head_dim)
dev = torch.device("cuda", 0)
q, k, v = make_inputs(cfg, dev)
flops = causal_flops(cfg["B"], cfg["Hq"], cfg["L"], cfg["d"])
runners = {}
for spec in a.libs:
    name, path = spec.split("=", 1)
    split = a.split
    if "@" in path:
        path, split = path.split("@")
        split = int(split)
    lib = _lib.bind(os.path.abspath(path))
    for pair in ((1, 2) if a.pair else (0,)):
        runners[name + ("" if pair == 0 else f"/pair{pair}")] = Runner(
            q, k, v, a.variant, lam=1e-2 if a.variant == "vsa" else None, k_block=a.k_block, lib=lib, cta_pair=pair)
        runners[name + ("" if pair == 0 else f"/pair{pair}")].p.softmax_split = split
sh = torch.cuda.current_stream().cuda_stream
for r in runners.values():
    for _ in range(3):
        r.krepr(sh)
        r.attn(sh)
torch.cuda.synchronize()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
clk = ClockSampler(0)
with clk:
    res = time_interleaved(runners, a.steps, flush, lambda: None)
first = next(iter(runners.values()))
for name, r in runners.items():
    same = torch.equal(r.o, first.o)
    print(f"{name:>12s}: attn {res[name][1]:.4f} ms  {flops / res[name][1] / 1e9:8.1f} TFLOP/s  "
          f"bitwise==first: {same}")
print("clocks", clk.summary())
