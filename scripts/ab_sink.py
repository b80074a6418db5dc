"""A/B of library builds on the C3 planted-sink problem (VSA at several lambdas).
    python scripts/ab_sink.py NAME=lib.so [NAME=lib.so ...]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, Runner, causal_flops, make_inputs, time_interleaved  # noqa: E402
from paper_2604_12798_b200 import _lib  # noqa: E402
from bench import planted_sink  # noqa: E402

cfg = dict(CONFIGS["c2"])
dev = torch.device("cuda", 0)
q, k, v = make_inputs(cfg, dev)
planted_sink(q, k, 8.0, 128)
flops = causal_flops(1, cfg["Hq"], cfg["L"], cfg["d"])
libs = [a.split("=", 1) for a in sys.argv[1:]]
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
for lam in (1e-4, 1e-3, 3e-3, 1e-2):
    runners = {name: Runner(q, k, v, "vsa", lam=lam, lib=_lib.bind(os.path.abspath(path))) for name, path in libs}
    sh = torch.cuda.current_stream().cuda_stream
    for r in runners.values():
        for _ in range(2):
            r.krepr(sh)
            r.attn(sh)
    torch.cuda.synchronize()
    res = time_interleaved(runners, 5, flush, lambda: None)
    first = next(iter(runners.values()))
    print(f"lam={lam:g} skipped={first.stats_dict()['skipped'] / first.stats_dict()['visited']:.3f} " +
          " ".join(f"{n}={flops / res[n][1] / 1e9:.0f}TF(eq={torch.equal(r.o, first.o)})" for n, r in runners.items()))
