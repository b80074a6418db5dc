"""One C2 forward of a chosen variant, for ncu captures (numbers printed under ncu are not bench values).

    ncu --set full -k regex:vfa_fwd_kernel -s 1 -c 1 -o prof python scripts/profile_step.py --variant vfa
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS, Runner, make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--variant", default="vfa", choices=("fa", "vfa", "vsa"))
ap.add_argument("--config", default="c2", choices=tuple(CONFIGS))
ap.add_argument("--lam", type=float, default=1e-2)
ap.add_argument("--k-block", type=int, default=128)
ap.add_argument("--head-dim", type=int, default=128)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--n-local", type=int, default=1)
ap.add_argument("--pair", type=int, default=0)
ap.add_argument("--split", type=int, default=0, help="softmax_split (0: per-variant default)")
ap.add_argument("--lib", default=None, help="experiment build (libvfa_b200_<name>.so) instead of the product library")
ap.add_argument("--stats-out", default=None, help="write the pass's block-class counts here (JSON)")
a = ap.parse_args()
cfg = dict(CONFIGS[a.config])
cfg["d"] = a.head_dim
dev = torch.device("cuda", 0)
q, k, v = make_inputs(cfg, dev)
lib = None
if a.lib:
    from paper_2604_12798_b200 import _lib
    lib = _lib.bind(os.path.abspath(a.lib))
r = Runner(q, k, v, a.variant, lam=a.lam if a.variant == "vsa" else None, k_block=a.k_block,
           n_local=a.n_local, cta_pair=a.pair, lib=lib)
r.p.softmax_split = a.split
sh = torch.cuda.current_stream().cuda_stream
for _ in range(a.iters):
    r.krepr(sh)
    r.attn(sh)
torch.cuda.synchronize()
print(a.variant, r.stats_dict())
if a.stats_out:
    import json
    with open(a.stats_out, "w") as f:
        json.dump(dict(variant=a.variant, d=a.head_dim, k_block=a.k_block, n_local=a.n_local, B=cfg["B"],
                       Hq=cfg["Hq"], Hkv=cfg["Hkv"], L=cfg["L"], stats=r.stats_dict()), f)
