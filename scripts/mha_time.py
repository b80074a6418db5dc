"""Time VFA / FA on MHA (Hq = Hkv, one query tile per CTA) vs GQA at the C2 size."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import Runner, causal_flops, time_interleaved  # noqa: E402
from paper_2604_12798_b200 import _lib  # noqa: E402

LIBS = [(a.split("=", 1)[0], _lib.bind(os.path.abspath(a.split("=", 1)[1]))) for a in sys.argv[1:]] or [
    ("lib", _lib.load())]


def run(hq, hkv, L=32768, d=128):
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    q = torch.randn((1, hq, L, d), generator=g, device=dev).to(torch.bfloat16)
    k = torch.randn((1, hkv, L, d), generator=g, device=dev).to(torch.bfloat16)
    v = torch.randn((1, hkv, L, d), generator=g, device=dev).to(torch.bfloat16)
    rs = {f"{name}@{tag}": Runner(q, k, v, name, lam=1e-2 if name == "vsa" else None, lib=lib)
          for name in ("vfa", "vsa", "fa") for tag, lib in LIBS}
    sh = torch.cuda.current_stream().cuda_stream
    for r in rs.values():
        for _ in range(2):
            r.krepr(sh)
            r.attn(sh)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    res = time_interleaved(rs, 5, flush, lambda: None)
    fl = causal_flops(1, hq, L, d)
    print(f"Hq={hq} Hkv={hkv}: " + " ".join(f"{n}={fl / res[n][1] / 1e9:.0f}TF" for n in rs))


run(32, 8)
run(32, 32)
run(24, 24)
