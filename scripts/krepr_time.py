"""Time the key-representation kernel alone at C2 (CUDA events, after warm-up)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, Runner, make_inputs  # noqa: E402

q, k, v = make_inputs(CONFIGS["c2"], torch.device("cuda", 0))
r = Runner(q, k, v, "vfa")
sh = torch.cuda.current_stream().cuda_stream
for _ in range(5):
    r.krepr(sh)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    r.krepr(sh)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 50 * 1e3
print(f"krepr: {us:.1f} us per launch, {k.numel() * 2 / (us * 1e-6) / 1e9:.0f} GB/s of K read")
