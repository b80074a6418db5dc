"""Per-kernel clock and work-per-cycle comparison (calibration, not bench values).

Each kernel runs back to back for ~1 s while NVML samples the SM clock; reported: TFLOP/s,
median SM MHz under load, and FLOP per SM-cycle (= TFLOP/s / (148 * MHz)), which separates
"runs at a lower clock under the power cap" from "does more work per cycle".

    python scripts/clock_efficiency.py [--only vfa,fa,vsa,cudnn,fa4] [--seconds 1.0]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, ClockSampler, Runner, _VendorRunner, causal_flops, make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--only", default="vfa,fa,cudnn,fa4")
ap.add_argument("--seconds", type=float, default=1.0)
ap.add_argument("--split", type=int, default=0)
a = ap.parse_args()
cfg = CONFIGS["c2"]
dev = torch.device("cuda", 0)
q, k, v = make_inputs(cfg, dev)
flops = causal_flops(cfg["B"], cfg["Hq"], cfg["L"], cfg["d"])
sh = torch.cuda.current_stream().cuda_stream
for name in a.only.split(","):
    try:
        if name in ("cudnn", "fa4"):
            r = _VendorRunner(name, q, k, v)
        else:
            r = Runner(q, k, v, name, lam=1e-2 if name == "vsa" else None)
            r.p.softmax_split = a.split
        for _ in range(3):
            r.krepr(sh)
            r.attn(sh)
        torch.cuda.synchronize()
        t0 = time.time()
        n = 0
        clk = ClockSampler(0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with clk:
            e0.record()
            while time.time() - t0 < a.seconds:
                for _ in range(10):
                    r.attn(sh)
                n += 10
                torch.cuda.synchronize()
            e1.record()
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        c = clk.summary()
        tf = flops / ms / 1e9
        mhz = c["sm_mhz"] or float("nan")
        print(f"{name:>6s}: {tf:8.1f} TFLOP/s  {ms:.4f} ms  SM {mhz:.0f} MHz  "
              f"{tf * 1e12 / (148 * mhz * 1e6):7.0f} FLOP/SM-cycle  reasons {c['reasons']}", flush=True)
        del r
        torch.cuda.empty_cache()
    except Exception as e:  # noqa: BLE001
        print(f"{name}: failed {type(e).__name__}: {str(e)[:200]}")
