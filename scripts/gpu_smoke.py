"""Quick GPU bring-up: run tiny FA/VFA/VSA cases and print errors vs the oracle."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import vfa_oracle as vo  # noqa: E402
from paper_2604_12798_b200 import attention_forward, stats_dict  # noqa: E402


def f64(t):
    return t.float().cpu().numpy().astype(np.float64)


def run(variant, L, d, bc, causal, hq=1, hkv=1, **extra):
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn((1, hq, L, d), generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn((1, hkv, L, d), generator=g, device="cuda").to(torch.bfloat16)
    v = torch.randn((1, hkv, L, d), generator=g, device="cuda").to(torch.bfloat16)
    kw = dict(variant=variant, causal=causal, q_block=128, k_block=bc, **extra)
    t0 = time.time()
    out, lse, info = attention_forward(q, k, v, check=False, **kw)
    torch.cuda.synchronize()
    st = stats_dict(info)
    ro, rl, rs = vo.forward(f64(q), f64(k), f64(v), **kw)
    o = f64(out)
    print(f"{kw} hq={hq} L={L} d={d}: O err {np.nanmax(np.abs(o - ro)):.3e} "
          f"rel {vo.max_rel_err(np.nan_to_num(o), ro):.3e} LSE err {np.nanmax(np.abs(lse.double().cpu().numpy() - rl)):.3e} "
          f"finite={np.isfinite(o).all()} st={st} ref={ {k2: rs[k2] for k2 in ('visited','skipped','special','frozen')} } "
          f"{time.time()-t0:.2f}s", flush=True)


if __name__ == "__main__":
    print(torch.cuda.get_device_name(), flush=True)
    run("fa", 128, 128, 128, False)
    run("fa", 256, 128, 128, True)
    run("vfa", 256, 128, 128, True, use_m_init=False)
    run("vfa", 512, 128, 128, True)
    run("fa", 512, 128, 128, True, hq=2)
    run("vfa", 512, 128, 128, True, hq=2)
    run("vsa", 512, 128, 128, True, hq=2, lam=1e-2)
    run("vfa", 512, 64, 64, True, hq=2)
    run("vfa", 512, 64, 128, False, hq=2)
    run("vfa", 512, 128, 64, True, hq=2, n_local=2)
