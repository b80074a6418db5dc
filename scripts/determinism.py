"""Run-to-run determinism of the default kernels at a given shape (development check).

    python scripts/determinism.py [--L 32768] [--hq 32] [--hkv 8] [--reps 3]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import make_inputs  # noqa: E402
from paper_2604_12798_b200 import attention_forward  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--L", type=int, default=32768)
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
q, k, v = make_inputs(dict(B=1, Hq=a.hq, Hkv=a.hkv, L=a.L, d=128), torch.device("cuda", 0))
for variant in ("vfa", "vsa", "fa"):
    outs = []
    for _ in range(a.reps):
        o, l, _ = attention_forward(q, k, v, variant=variant, causal=True, check=False,
                                    lam=1e-2 if variant == "vsa" else None)
        outs.append((o.clone(), l.clone()))
    torch.cuda.synchronize()
    same = all(torch.equal(outs[0][0], x[0]) and torch.equal(outs[0][1], x[1]) for x in outs[1:])
    ndiff = max(int((outs[0][0] != x[0]).sum()) for x in outs[1:])
    qh, kh, vh = (x.cpu().pin_memory() for x in (q, k, v))
    h = attention_forward(qh, kh, vh, variant=variant, causal=True, lam=1e-2 if variant == "vsa" else None)
    do = (h[0] != outs[0][0].cpu())
    hs = (not bool(do.any())) and torch.equal(h[1], outs[0][1].cpu())
    where = ""
    if do.any():
        idx = do.nonzero()
        heads = sorted(set(idx[:, 1].tolist()))
        rows = idx[:, 2]
        dl = (h[1] != outs[0][1].cpu()).nonzero()
        where = (f" differing O elements {int(do.sum())} in heads {heads[:8]} rows {int(rows.min())}..{int(rows.max())};"
                 f" LSE rows differing {dl.shape[0]}")
    print(f"{variant}: deterministic {same} (max differing O elements {ndiff}); host pipeline bitwise {hs}{where}")
