"""BASELINE.json configs[2] (C3: VSA lambda sweep) and configs[4] (C5: Bc x d ablation) at full
step counts (bench.py's default line carries the same sweeps at 5 steps).

    python scripts/sweeps.py c3 [--steps 10]   # planted-sink data at the C2 shape, lambda sweep
    python scripts/sweeps.py c5 [--steps 10]   # Bc in {64,128} x d in {64,128}, FA vs VFA
Prints one JSON object. TFLOP/s are algorithmic (dense-equivalent) causal FLOPs / attention-kernel
time; for VSA that is the "effective" rate (skipped blocks still count).
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, ClockSampler, c3_sweep, c5_ablation, planted_sink  # noqa: E402,F401

ap = argparse.ArgumentParser()
ap.add_argument("which", choices=("c3", "c5"))
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
dev = torch.device("cuda", 0)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
clk = ClockSampler(0)
with clk:
    res = (c3_sweep if a.which == "c3" else c5_ablation)(dict(CONFIGS["c2"]), dev, flush, a.steps)
print(json.dumps({"config": a.which.upper(), "result": res, "clocks": clk.summary()}))
