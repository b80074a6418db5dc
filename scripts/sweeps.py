"""BASELINE.json configs[2] (C3: VSA lambda sweep) and configs[4] (C5: Bc x d ablation).

    python scripts/sweeps.py c3     # planted-sink data at the C2 shape, lambda sweep
    python scripts/sweeps.py c5     # Bc in {64,128} x d in {64,128}, FA vs VFA
Prints one JSON object per line. TFLOP/s are algorithmic (dense-equivalent) causal FLOPs /
attention-kernel time; for VSA that is the "effective" rate (skipped blocks still count).
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, ClockSampler, Runner, causal_flops, make_inputs, time_interleaved  # noqa: E402


def planted_sink(q, k, boost, bc):
    d = q.shape[-1]
    amp = float(np.sqrt(boost * np.sqrt(d)))
    q[..., 0] = amp
    k[..., 0] = 0
    k[:, :, :bc, 0] = amp


def run_c3():
    from oracle import vfa_oracle as vo
    cfg = dict(CONFIGS["c2"])
    dev = torch.device("cuda", 0)
    q, k, v = make_inputs(cfg, dev)
    planted_sink(q, k, 8.0, 128)
    flops = causal_flops(1, cfg["Hq"], cfg["L"], cfg["d"])
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    base = Runner(q, k, v, "vfa")
    runners = {"vfa": base}
    lams = (1e-4, 1e-3, 3e-3, 1e-2, 3e-2, 1e-1)
    for lam in lams:
        runners[f"vsa_{lam:g}"] = Runner(q, k, v, "vsa", lam=lam)
    sh = torch.cuda.current_stream().cuda_stream
    for r in runners.values():
        for _ in range(3):
            r.krepr(sh)
            r.attn(sh)
    torch.cuda.synchronize()
    timed = time_interleaved(runners, 10, flush, lambda: None)
    ref_o = base.o.float()
    # oracle on sampled query blocks of head 0 (float64, identical bf16 inputs)
    qb = [1, 64, 128, 200, 256]
    q0 = q[0, 0].double().cpu().numpy()
    k0, v0 = k[0, 0].double().cpu().numpy(), v[0, 0].double().cpu().numpy()
    for name, r in runners.items():
        st = r.stats_dict()
        line = {"config": "C3", "variant": name, "attn_kernel_ms": round(timed[name][1], 4),
                "effective_tflops": round(flops / timed[name][1] / 1e9, 1),
                "skipped_fraction": round(st["skipped"] / max(st["visited"], 1), 4), **st}
        o = r.o.float()
        line["max_abs_vs_vfa"] = float((o - ref_o).abs().max())
        if name != "vfa":
            lam = float(name.split("_")[1])
            res = vo.forward_head(q0, k0, v0, variant="vsa", causal=True, q_block=128, k_block=128,
                                  lam=lam, q_blocks=qb)
            rows = np.concatenate([np.arange((i - 1) * 128, i * 128) for i in qb])
            got = r.o[0, 0].double().cpu().numpy()[rows]
            line["oracle_rows"] = len(rows)
            line["max_abs_vs_oracle"] = float(np.abs(got - res.out[rows]).max())
            line["max_rel_err_vs_oracle"] = vo.max_rel_err(got, res.out[rows])
            line["oracle_skipped_in_sample"] = res.skipped
        print(json.dumps(line), flush=True)


def run_c5():
    dev = torch.device("cuda", 0)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    for d in (64, 128):
        cfg = dict(CONFIGS["c2"], d=d)
        q, k, v = make_inputs(cfg, dev)
        flops = causal_flops(1, cfg["Hq"], cfg["L"], d)
        for bc in (64, 128):
            nl = 2 if bc == 64 else 1
            runners = {"fa": Runner(q, k, v, "fa", k_block=bc, n_local=nl),
                       "vfa": Runner(q, k, v, "vfa", k_block=bc, n_local=nl)}
            sh = torch.cuda.current_stream().cuda_stream
            for r in runners.values():
                for _ in range(3):
                    r.krepr(sh)
                    r.attn(sh)
            torch.cuda.synchronize()
            clk = ClockSampler(0)
            with clk:
                timed = time_interleaved(runners, 10, flush, lambda: None)
            line = {"config": "C5", "head_dim": d, "k_block": bc, "n_local": nl, "clocks": clk.summary()}
            for name in runners:
                line[f"{name}_tflops"] = round(flops / timed[name][1] / 1e9, 1)
            line["vfa_speedup"] = round(timed["fa"][1] / timed["vfa"][1], 4)
            print(json.dumps(line), flush=True)
        del q, k, v


if __name__ == "__main__":
    {"c3": run_c3, "c5": run_c5}[sys.argv[1]]()
