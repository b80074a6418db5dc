"""Timeline of the host-resident pipeline (vfa_fwd_host) on the C2 problem.

    VFA_HOST_TIMELINE=1 python scripts/host_timeline.py [--chunk 1] [--qchunk 2]
The library prints per-stage CUDA-event times (debug mode, synchronizing); this script runs
the pipeline twice (warm-up, then recorded) and summarises fill, steady state and drain.
"""
import argparse
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if os.environ.get("_VFA_TL_CHILD"):
    import torch
    sys.path.insert(0, ROOT)
    from bench import CONFIGS, make_inputs  # noqa: E402
    from paper_2604_12798_b200 import attention_forward_host  # noqa: E402
    ck, cq, n = (int(x) for x in sys.argv[1:4])
    cfg = CONFIGS["c2"]
    q, k, v = (x.cpu().pin_memory() for x in make_inputs(cfg, torch.device("cuda", 0)))
    for i in range(n):
        if i == n - 1:
            sys.stderr.write("vfa_host_timeline RUN\n")
        attention_forward_host(q, k, v, variant="vfa", causal=True, chunk_kv_heads=ck, chunk_q_heads=cq)
        torch.cuda.synchronize()
    sys.exit(0)

ap = argparse.ArgumentParser()
ap.add_argument("--chunk", type=int, default=1)
ap.add_argument("--qchunk", type=int, default=2)
a = ap.parse_args()
env = dict(os.environ, VFA_HOST_TIMELINE="1", _VFA_TL_CHILD="1")
out = subprocess.run([sys.executable, __file__, str(a.chunk), str(a.qchunk), "3"], env=env,
                     capture_output=True, text=True).stderr.splitlines()
lines = [ln.split() for ln in out if ln.startswith("vfa_host_timeline")]
if not any(ln[1] == "RUN" for ln in lines):
    sys.exit("child failed:\n" + "\n".join(out[-20:]))
last = max(i for i, ln in enumerate(lines) if ln[1] == "RUN")
ev = {}
for ln in lines[last + 1:]:
    name = " ".join(ln[1:-3])
    ev[name] = float(ln[-3])
chunks = sorted({int(k.split()[1]) for k in ev if k.startswith("q_in")})
print(f"chunks {len(chunks)}; total {max(ev.values()):.3f} ms")
print(f"{'chunk':>5} {'q_in':>8} {'k_start':>8} {'k_end':>8} {'out':>8}  kernel ms")
for c in chunks:
    print(f"{c:5d} {ev[f'q_in {c}']:8.3f} {ev[f'k_start {c}']:8.3f} {ev[f'k_end {c}']:8.3f} {ev[f'out {c}']:8.3f}"
          f"  {ev[f'k_end {c}'] - ev[f'k_start {c}']:.3f}")
first_k = min(ev[f"k_start {c}"] for c in chunks)
last_in = max(ev[f"q_in {c}"] for c in chunks)
last_k = max(ev[f"k_end {c}"] for c in chunks)
print(f"fill (entry -> first kernel) {first_k:.3f} ms; last H2D {last_in:.3f}; last kernel end {last_k:.3f}; "
      f"drain (last H2D -> end) {max(ev.values()) - last_in:.3f}")
