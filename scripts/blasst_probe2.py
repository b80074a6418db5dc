import sys, torch
sys.path.insert(0, '.')
from paper_2604_12798_b200 import attention_forward, stats_dict
g = torch.Generator(device='cuda').manual_seed(0)
q = torch.randn((1, 4, 1024, 128), generator=g, device='cuda').to(torch.bfloat16)
k = torch.randn((1, 2, 1024, 128), generator=g, device='cuda').to(torch.bfloat16)
v = torch.randn((1, 2, 1024, 128), generator=g, device='cuda').to(torch.bfloat16)
for split in (2, 4):
    o0, l0, _ = attention_forward(q, k, v, variant="fa", causal=True, softmax_split=split)
    for var in ("blasst", "blasst_rowskip", "blasst_fa4"):
        o1, l1, i1 = attention_forward(q, k, v, variant=var, causal=True, softmax_split=split, lam=None)
        d = (o1.float() - o0.float()).abs()
        idx = (d > 0).nonzero()
        print(split, var, "O maxdiff", d.max().item(), "n diff", idx.shape[0], "LSE maxdiff", (l1 - l0).abs().max().item(),
              "first", idx[:3].tolist(), stats_dict(i1))
