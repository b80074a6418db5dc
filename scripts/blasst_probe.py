import sys, torch
sys.path.insert(0, '.')
from paper_2604_12798_b200 import attention_forward, stats_dict
variant = sys.argv[1]; d = int(sys.argv[2]); bc = int(sys.argv[3]); split = int(sys.argv[4])
g = torch.Generator(device='cuda').manual_seed(0)
q = torch.randn((1, 4, 1024, d), generator=g, device='cuda').to(torch.bfloat16)
k = torch.randn((1, 2, 1024, d), generator=g, device='cuda').to(torch.bfloat16)
v = torch.randn((1, 2, 1024, d), generator=g, device='cuda').to(torch.bfloat16)
o, l, info = attention_forward(q, k, v, variant=variant, causal=True, k_block=bc, lam=1e-2, tau=2.0, softmax_split=split, check=False)
torch.cuda.synchronize()
print(variant, d, bc, split, 'ok', stats_dict(info))
