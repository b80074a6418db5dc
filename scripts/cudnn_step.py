"""One cuDNN fused-attention forward at the C2 shape (K/V expanded), for ncu captures (calibration)."""
import torch
import torch.nn.functional as F
from torch.nn.attention import SDPBackend, sdpa_kernel

B, Hq, Hkv, L, d = 1, 32, 8, 32768, 128
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
q = torch.randn(B, Hq, L, d, generator=g, device=dev, dtype=torch.bfloat16)
k = torch.randn(B, Hkv, L, d, generator=g, device=dev, dtype=torch.bfloat16).repeat_interleave(Hq // Hkv, dim=1)
v = torch.randn(B, Hkv, L, d, generator=g, device=dev, dtype=torch.bfloat16).repeat_interleave(Hq // Hkv, dim=1)
with sdpa_kernel(SDPBackend.CUDNN_ATTENTION):
    for _ in range(3):
        o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
torch.cuda.synchronize()
