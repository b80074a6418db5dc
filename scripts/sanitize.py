"""Small forward of every variant / layout for compute-sanitizer (SURVEY.md §5 race detection).

    compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python scripts/sanitize.py
Each launch covers a causal and a non-causal problem at (d, Bc) in {(128,128), (64,64)}, with
GQA, every variant, the softmax layouts, CTA pairs, the block-wise query seeds and the host
pipeline. Prints one line per case; the sanitizer's own summary is the verdict.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_12798_b200 import attention_forward, attention_forward_host  # noqa: E402


def rand(shape, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(shape, generator=g, device="cuda").to(torch.bfloat16)


L = int(os.environ.get("SAN_L", "256"))
cases = []
for variant in ("fa", "vfa", "vsa", "blasst", "blasst_fa4", "blasst_rowskip"):
    for d, bc in ((128, 128), (64, 64)):
        for causal in (True, False):
            kw = dict(variant=variant, causal=causal, k_block=bc, lam=1e-2 if variant not in ("fa", "vfa") else None)
            if variant == "blasst_fa4":
                kw["tau"] = 2.0
            cases.append((d, kw))
for split in (1, 2, 4):
    cases.append((128, dict(variant="vfa", causal=True, softmax_split=split)))
cases.append((128, dict(variant="vfa", causal=True, cta_pair=2)))
cases.append((128, dict(variant="vsa", causal=True, cta_pair=2, lam=1e-2)))
cases.append((128, dict(variant="vfa", causal=True, qkind="q_mean")))
cases.append((128, dict(variant="vfa", causal=True, q_block=64, k_block=64)))
cases.append((128, dict(variant="vfa", causal=True, monitor=True)))
for i, (d, kw) in enumerate(cases):
    q, k, v = rand((1, 4, L, d), 3 * i), rand((1, 1, L, d), 3 * i + 1), rand((1, 1, L, d), 3 * i + 2)
    out, lse, info = attention_forward(q, k, v, check=False, **kw)
    torch.cuda.synchronize()
    print("ok", d, kw, bool(torch.isfinite(out).all()), flush=True)
q, k, v = rand((1, 8, L, 128), 90), rand((1, 2, L, 128), 91), rand((1, 2, L, 128), 92)
o, l, _ = attention_forward_host(q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory(), variant="vfa",
                                 causal=True, qkind="q_absmax", chunk_kv_heads=1, chunk_q_heads=2)
print("ok host pipeline", bool(torch.isfinite(o).all()), flush=True)
