"""Calibration (not the product): this repo's VFA / FA kernels against vendor attention
kernels on the C2 problem, timed interleaved step by step in one process, L2 flushed before
every step (same protocol as bench.py):
  cudnn  torch SDPA, cuDNN backend (K/V expanded to the query heads)
  fa4    the FlashAttention-4 CuTe-DSL forward shipped inside vllm (vllm_flash_attn.cute),
         native GQA, [B, L, H, d] layout (inputs transposed once, outside the timed region)

    python scripts/vs_vendor.py [--steps 20] [--only vfa,fa,cudnn,fa4]
"""
import argparse
import os
import sys

import torch
import torch.nn.functional as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, ClockSampler, Runner, causal_flops, make_inputs, time_interleaved  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--only", default="vfa,fa,cudnn,fa4")
ap.add_argument("--config", default="c2")
a = ap.parse_args()
cfg = CONFIGS[a.config]
dev = torch.device("cuda", 0)
q, k, v = make_inputs(cfg, dev)
flops = causal_flops(cfg["B"], cfg["Hq"], cfg["L"], cfg["d"])
rep = cfg["Hq"] // cfg["Hkv"]


class Cudnn:
    def __init__(self):
        self.ke, self.ve = (x.repeat_interleave(rep, dim=1) for x in (k, v))

    def krepr(self, stream):
        pass

    def attn(self, stream):
        from torch.nn.attention import SDPBackend, sdpa_kernel
        with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
            self.o = F.scaled_dot_product_attention(q, self.ke, self.ve, is_causal=True)


class FA4:
    def __init__(self):
        from vllm.vllm_flash_attn.cute import flash_attn_func
        self.f = flash_attn_func
        self.qt, self.kt, self.vt = (x.transpose(1, 2).contiguous() for x in (q, k, v))

    def krepr(self, stream):
        pass

    def attn(self, stream):
        out = self.f(self.qt, self.kt, self.vt, causal=True)
        self.o = (out[0] if isinstance(out, tuple) else out).transpose(1, 2)


makers = {"vfa": lambda: Runner(q, k, v, "vfa"), "fa": lambda: Runner(q, k, v, "fa"), "cudnn": Cudnn, "fa4": FA4}
runners = {}
for name in a.only.split(","):
    try:
        runners[name] = makers[name]()
    except Exception as e:  # calibration only: report and go on
        print(f"{name}: unavailable ({type(e).__name__}: {e})")
sh = torch.cuda.current_stream().cuda_stream
for name in list(runners):
    try:
        for _ in range(3):
            runners[name].krepr(sh)
            runners[name].attn(sh)
        torch.cuda.synchronize()
    except Exception as e:
        print(f"{name}: failed ({type(e).__name__}: {str(e)[:300]})")
        del runners[name]
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
clk = ClockSampler(0)
with clk:
    res = time_interleaved(runners, a.steps, flush, lambda: None)
for name in runners:
    print(f"{name:>6s}: attention {res[name][1]:.4f} ms  {flops / res[name][1] / 1e9:8.1f} TFLOP/s")
if "vfa" in runners:
    o_ref = runners["vfa"].o.float()
    for name in runners:
        if name != "vfa":
            print(f"max |O_{name} - O_vfa| =", (runners[name].o.float() - o_ref).abs().max().item())
print("clocks", clk.summary())
