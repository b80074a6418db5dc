"""Calibration only (not the product): time library attention kernels at the C2 shape to
know what this B200 reaches with vendor code. torch SDPA (cuDNN / flash backends) and
FlashInfer's prefill if importable."""
import time

import torch
import torch.nn.functional as F

B, Hq, Hkv, L, d = 1, 32, 8, 32768, 128
flops = 4.0 * B * Hq * L * L * d / 2
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
q = torch.randn(B, Hq, L, d, generator=g, device=dev, dtype=torch.bfloat16)
k = torch.randn(B, Hkv, L, d, generator=g, device=dev, dtype=torch.bfloat16)
v = torch.randn(B, Hkv, L, d, generator=g, device=dev, dtype=torch.bfloat16)


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402
for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
    try:
        with sdpa_kernel(be):
            ms = timeit(lambda: F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True))
        print(f"sdpa[{name}] {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"sdpa[{name}] unavailable: {str(e).splitlines()[0][:120]}", flush=True)
# cuDNN without the GQA flag: K / V expanded to the query heads
ke, ve = (x.repeat_interleave(Hq // Hkv, dim=1) for x in (k, v))
for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION),):
    try:
        with sdpa_kernel(be):
            ms = timeit(lambda: F.scaled_dot_product_attention(q, ke, ve, is_causal=True))
        print(f"sdpa[{name}, K/V expanded] {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"sdpa[{name}, K/V expanded] unavailable: {str(e).splitlines()[0][:120]}", flush=True)
try:
    import flashinfer
    qf = q[0].transpose(0, 1).contiguous()  # [L, Hq, d]
    kf = k[0].transpose(0, 1).contiguous()
    vf = v[0].transpose(0, 1).contiguous()
    for backend in ("cutlass", "fa3", "fa2", "auto"):
        try:
            ms = timeit(lambda: flashinfer.single_prefill_with_kv_cache(qf, kf, vf, causal=True, backend=backend))
            print(f"flashinfer[{backend}] {ms:.3f} ms  {flops / ms / 1e9:.1f} TFLOP/s", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"flashinfer[{backend}] unavailable: {str(e).splitlines()[0][:120]}", flush=True)
except Exception as e:  # noqa: BLE001
    print("flashinfer unavailable:", str(e).splitlines()[0][:120])
