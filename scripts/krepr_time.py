"""Time the key-representation kernel alone at C2 (CUDA events): cold (L2 flushed before each
launch, K streamed from HBM -- the bench's situation) and hot (back to back, K L2-resident)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, Runner, make_inputs  # noqa: E402

q, k, v = make_inputs(CONFIGS["c2"], torch.device("cuda", 0))
lib = None
if len(sys.argv) > 1:
    from paper_2604_12798_b200 import _lib
    lib = _lib.bind(os.path.abspath(sys.argv[1]))
r = Runner(q, k, v, "vfa", lib=lib)
sh = torch.cuda.current_stream().cuda_stream
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=q.device)
for _ in range(5):
    r.krepr(sh)
cold = []
for _ in range(20):
    flush.fill_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r.krepr(sh)
    e1.record()
    torch.cuda.synchronize()
    cold.append(e0.elapsed_time(e1) * 1e3)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    r.krepr(sh)
e1.record()
torch.cuda.synchronize()
hot = e0.elapsed_time(e1) / 50 * 1e3
cold.sort()
c = cold[len(cold) // 2]
nbytes = k.numel() * 2 + r.ws_bytes
print(f"krepr: cold {c:.1f} us ({nbytes / (c * 1e-6) / 1e9:.0f} GB/s of K read + reprs written), "
      f"hot {hot:.1f} us ({nbytes / (hot * 1e-6) / 1e9:.0f} GB/s)")
