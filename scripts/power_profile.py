"""Calibration (not the product): sustained throughput, SM clock and board power of this repo's
attention kernels and of vendor kernels on the C2 problem. Each kernel runs back to back for
`--seconds` while NVML samples the SM clock and power; the report gives TFLOP/s, median clock,
median power, TFLOP/s per GHz (tensor-pipe utilisation proxy) and TFLOP per joule (energy
efficiency). Under the B200's power cap these two separate "idle cycles" from "energy per FLOP".

    python scripts/power_profile.py [--seconds 3] [--only vfa,fa,vsa,cudnn,fa4] [--lib path@split ...]
"""
import argparse
import os
import sys
import threading
import time

import numpy as np
import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, Runner, causal_flops, make_inputs  # noqa: E402
from paper_2604_12798_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=3.0)
ap.add_argument("--only", default="vfa,fa,vsa,cudnn,fa4")
ap.add_argument("--lib", action="append", default=[], help="NAME=path.so[@split][:variant] extra builds")
ap.add_argument("--config", default="c2")
a = ap.parse_args()
cfg = CONFIGS[a.config]
dev = torch.device("cuda", 0)
q, k, v = make_inputs(cfg, dev)
flops = causal_flops(cfg["B"], cfg["Hq"], cfg["L"], cfg["d"])
rep = cfg["Hq"] // cfg["Hkv"]


def cudnn():
    ke, ve = (x.repeat_interleave(rep, dim=1) for x in (k, v))
    from torch.nn.attention import SDPBackend, sdpa_kernel

    def f():
        with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
            F.scaled_dot_product_attention(q, ke, ve, is_causal=True)
    return f


def fa4():
    from vllm.vllm_flash_attn.cute import flash_attn_func
    qt, kt, vt = (x.transpose(1, 2).contiguous() for x in (q, k, v))
    return lambda: flash_attn_func(qt, kt, vt, causal=True)


def ours(variant, lib=None, split=0):
    r = Runner(q, k, v, variant, lam=1e-2 if variant == "vsa" else None, lib=lib)
    r.p.softmax_split = split
    sh = torch.cuda.current_stream().cuda_stream

    def f():
        r.krepr(sh)
        r.attn(sh)
    return f


makers = {"vfa": lambda: ours("vfa"), "fa": lambda: ours("fa"), "vsa": lambda: ours("vsa"), "cudnn": cudnn, "fa4": fa4}
fns = {}
for name in a.only.split(","):
    try:
        fns[name] = makers[name]()
    except Exception as e:
        print(f"{name}: unavailable ({type(e).__name__}: {e})")
for spec in a.lib:
    name, path = spec.split("=", 1)
    variant, split = "vfa", 0
    if ":" in path:
        path, variant = path.split(":")
    if "@" in path:
        path, split = path.split("@")
        split = int(split)
    fns[name] = ours(variant, _lib.bind(os.path.abspath(path)), split)

import pynvml  # noqa: E402
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


def measure(f):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    # calibrate the launch count for ~seconds
    t0 = time.perf_counter()
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    per = (time.perf_counter() - t0) / 5
    n = max(5, int(a.seconds / per))
    clk, pw = [], []
    stop = threading.Event()

    def sample():
        while not stop.is_set():
            clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
            time.sleep(0.02)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    th = threading.Thread(target=sample, daemon=True)
    th.start()
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / n
    # drop the first quarter of the samples (power ramp)
    c = np.array(clk[len(clk) // 4:])
    p = np.array(pw[len(pw) // 4:])
    return ms, float(np.median(c)), float(np.median(p))


for name, f in fns.items():
    try:
        ms, mhz, watts = measure(f)
    except Exception as e:
        print(f"{name}: failed ({type(e).__name__}: {str(e)[:200]})")
        continue
    tf = flops / ms / 1e9
    print(f"{name:>10s}: {ms:7.3f} ms  {tf:7.1f} TFLOP/s  sm {mhz:6.0f} MHz  {watts:6.1f} W  "
          f"{tf / (mhz / 1000):6.1f} TFLOP/s/GHz  {tf / watts:5.3f} TFLOP/J")
    time.sleep(1.0)
