"""Calibration (not the product): this repo's VFA / FA kernels and cuDNN's fused attention
(torch SDPA, cuDNN backend, K/V expanded to the query heads) timed interleaved step by step in
one process on the C2 problem, L2 flushed before every step (same protocol as bench.py).

    python scripts/vs_cudnn.py [--steps 20]
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
a = ap.parse_args()
cfg = CONFIGS["c2"]
dev = torch.device("cuda", 0)
q, k, v = make_inputs(cfg, dev)
flops = causal_flops(cfg["B"], cfg["Hq"], cfg["L"], cfg["d"])
rep = cfg["Hq"] // cfg["Hkv"]
ke, ve = (x.repeat_interleave(rep, dim=1) for x in (k, v))


class Cudnn:
    def krepr(self, stream):
        pass

    def attn(self, stream):
        from torch.nn.attention import SDPBackend, sdpa_kernel
        with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
            self.o = F.scaled_dot_product_attention(q, ke, ve, is_causal=True)


runners = {"vfa": Runner(q, k, v, "vfa"), "fa": Runner(q, k, v, "fa"), "cudnn": Cudnn()}
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
for name in runners:
    print(f"{name:>6s}: attention {res[name][1]:.4f} ms  {flops / res[name][1] / 1e9:8.1f} TFLOP/s")
o_ref = runners["cudnn"].o.float()
print("max |O_vfa - O_cudnn| =", (runners["vfa"].o.float() - o_ref).abs().max().item(),
      " max |O_fa - O_cudnn| =", (runners["fa"].o.float() - o_ref).abs().max().item())
print("clocks", clk.summary())
