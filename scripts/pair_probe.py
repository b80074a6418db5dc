"""Probe the CTA-pair path (cta_pair=2) against the single-CTA path on small problems."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_12798_b200 import attention_forward, stats_dict  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
for variant in sys.argv[1:] or ["vfa"]:
    for L, bc in ((512, 128), (1024, 128), (1024, 64)):
        q = torch.randn((1, 4, L, 128), generator=g, device="cuda").to(torch.bfloat16)
        k = torch.randn((1, 2, L, 128), generator=g, device="cuda").to(torch.bfloat16)
        v = torch.randn((1, 2, L, 128), generator=g, device="cuda").to(torch.bfloat16)
        kw = dict(variant=variant, causal=True, k_block=bc, check=False, lam=1e-2 if variant != "vfa" else None)
        o1, l1, i1 = attention_forward(q, k, v, cta_pair=1, softmax_split=4, **kw)
        o2, l2, i2 = attention_forward(q, k, v, cta_pair=2, **kw)
        torch.cuda.synchronize()
        print(variant, L, bc, "O maxdiff", (o1.float() - o2.float()).abs().max().item(), "LSE maxdiff",
              (l1 - l2).abs().max().item(), "bitwise", torch.equal(o1, o2), stats_dict(i1) == stats_dict(i2), flush=True)
