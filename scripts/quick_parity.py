"""Quick GPU parity check of one library build against the CPU oracle (development aid).

    VFA_B200_LIB=path.so python scripts/quick_parity.py [--L 1024] [--hq 4] [--hkv 2]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import vfa_oracle as vo  # noqa: E402  (checker)
from paper_2604_12798_b200 import attention_forward, stats_dict  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--L", type=int, default=1024)
ap.add_argument("--hq", type=int, default=4)
ap.add_argument("--hkv", type=int, default=2)
ap.add_argument("--b", type=int, default=1)
a = ap.parse_args()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
q = torch.randn((a.b, a.hq, a.L, 128), generator=g, device=dev).to(torch.bfloat16)
k = torch.randn((a.b, a.hkv, a.L, 128), generator=g, device=dev).to(torch.bfloat16)
v = torch.randn((a.b, a.hkv, a.L, 128), generator=g, device=dev).to(torch.bfloat16)
f64 = lambda t: t.float().cpu().numpy().astype(np.float64)  # noqa: E731
for variant, kw in (("vfa", {}), ("fa", {}), ("vsa", {"lam": 1e-2}), ("vfa", {"reorder": False})):
    out, lse, info = attention_forward(q, k, v, variant=variant, causal=True, check=False, **kw)
    torch.cuda.synchronize()
    st = stats_dict(info)
    ro, rl, rst = vo.forward(f64(q), f64(k), f64(v), variant=variant, causal=True, q_block=128, k_block=128, **kw)
    err = float(np.abs(f64(out) - ro).max())
    rel = vo.max_rel_err(f64(out), ro)
    lerr = float(np.abs(lse.double().cpu().numpy() - rl).max())
    ok = err <= 2e-2 and rel <= 1e-2 and lerr <= 1e-4
    print(f"{variant} {kw}: O max abs {err:.3e} rel {rel:.3e} LSE {lerr:.3e} stats {st} ref "
          f"{ {k2: rst[k2] for k2 in ('visited', 'skipped', 'special', 'frozen') if k2 in rst} } {'OK' if ok else 'FAIL'}")
