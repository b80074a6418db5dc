"""Per-visit timeline of CTA 0 (the longest causal unit) from the debug trace.

    python scripts/trace_timeline.py [--variant vfa|fa|vsa] [--k-block 128]
Prints, per query tile, the softmax busy time per block (S ready -> P done), the gap the
softmax waits for the next S, the MMA's latency to observe P, and the per-block period.
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_12798_b200 import _lib, build  # noqa: E402

# the -DVFA_TRACE variant of the library (VFA_TRACE_LIB: an experiment build made with
# build.build(trace=True, defines=(name, flags)))
_lib.LIB_PATH = os.environ.get("VFA_TRACE_LIB") or build.build(trace=True)
from bench import CONFIGS, Runner, make_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--variant", default="vfa")
ap.add_argument("--k-block", type=int, default=128)
ap.add_argument("--n-local", type=int, default=1)
ap.add_argument("--sink", type=float, default=0.0, help="planted-sink boost (C3 data); 0 = Gaussian")
ap.add_argument("--lam", type=float, default=1e-2)
ap.add_argument("--pair", type=int, default=0, help="cta_pair (2 = CTA pairs)")
ap.add_argument("--split", type=int, default=0, help="softmax_split (0: per-variant default)")
ap.add_argument("--ws1", action="store_true", help="the decoupled one-tile kernel's slot layout")
ap.add_argument("--seq", type=int, default=0, help="sequence length override (C2 heads / head dim)")
a = ap.parse_args()
cfg = dict(CONFIGS["c2"])
if a.seq:
    cfg["L"] = a.seq
dev = torch.device("cuda", 0)
q, k, v = make_inputs(cfg, dev)
if a.sink:
    from bench import planted_sink
    planted_sink(q, k, a.sink, a.k_block)
r = Runner(q, k, v, a.variant, lam=a.lam if a.variant == "vsa" else None, k_block=a.k_block, n_local=a.n_local,
           cta_pair=a.pair)
r.p.softmax_split = a.split
T = cfg["L"] // a.k_block
# CTAs: one per unit (two heads); CTA pairs cover four heads per cluster when the group allows
units = cfg["B"] * cfg["Hkv"] * (cfg["L"] // 128) * (cfg["Hq"] // cfg["Hkv"] // 2)
if a.ws1:
    units *= 2  # one CTA per query tile
NS_ = 32  # vfa_kernel.cuh kTraceSlots
buf = torch.zeros(T * NS_ + units * 4, dtype=torch.int64, device=dev)
sh = torch.cuda.current_stream().cuda_stream
r.krepr(sh)
r.attn(sh)  # warm-up
r.lib.vfa_debug_trace(buf.data_ptr())
r.krepr(sh)
r.attn(sh)
torch.cuda.synchronize()
r.lib.vfa_debug_trace(None)
allbuf = buf.cpu().numpy()
ut = allbuf[T * NS_:].reshape(units, 4).astype(np.float64)
ok = (ut > 0).all(axis=1)
ut = ut[ok]
dur = ut[:, 3] - ut[:, 0]
pro = ut[:, 1] - ut[:, 0]
epi = ut[:, 3] - ut[:, 2]
print(f"units {ok.sum()}: mean cycles {dur.mean():.0f}; prologue (entry -> first S) {pro.mean():.0f} "
      f"({pro.sum() / dur.sum():.1%}), epilogue (last P -> exit) {epi.mean():.0f} ({epi.sum() / dur.sum():.1%})")
tr = allbuf[: T * NS_].reshape(T, NS_).astype(np.float64)
n = int((tr[:, 1] > 0).sum())
tr = tr[:n]
t0 = tr[tr > 0].min()
tr = np.where(tr > 0, tr - t0, np.nan)
if a.ws1:
    sl = slice(4, n - 4)
    print(f"variant={a.variant} visited={n} total={np.nanmax(tr):.0f} cycles -> {np.nanmax(tr) / n:.0f} cycles per block")
    S, P, P0, E, seen0, qk, pv, vacq, seen1 = (tr[:, i] for i in (0, 1, 2, 3, 4, 5, 6, 7, 8))
    med = lambda x: np.nanmedian(x[sl])  # noqa: E731
    print(f" softmax: waits for S {med(S - E):.0f}; S -> chunk-0 P {med(P0 - S):.0f}; S -> P done {med(P - S):.0f};"
          f" per-group period (pos -> pos+2) {med(S[2:] - S[:-2]):.0f}; next S after P done {med(S[2:] - P[:-2]):.0f}")
    print(f" MMA: V acquired {med(vacq - P0):.0f} after chunk-0 P; sees chunk 0 +{med(seen0 - P0):.0f}, chunk 1 +{med(seen1 - P):.0f};"
          f" PV issued +{med(pv - P):.0f} after P done; QK(g+3) issued +{med(qk - pv):.0f} after PV;"
          f" PV period {med(np.diff(pv)):.0f}")
    Ktma, Vtma, Kacq, bfree, mx, dec = (tr[:, i] for i in (11, 12, 13, 14, 9, 10))
    print(f" QK: buffer free (PV(g-3) issued) -> K acquired {med(Kacq - bfree):.0f}; K TMA issue -> K acquired"
          f" {med(Kacq - Ktma):.0f}; K TMA issued {med(Ktma - bfree):.0f} after buffer free; K acquired -> S ready"
          f" {med(S - Kacq):.0f}")
    print(f" V: TMA issue -> V acquired {med(vacq - Vtma):.0f}; V TMA issued {med(Vtma - S):.0f} after S ready")
    print(f" S (first chunk) in registers {med(tr[:, 15] - S):.0f} after S ready")
    qk_end = np.concatenate([qk[3:], np.full(3, np.nan)])  # QK(p) enqueued (slot 5 of element p - 3)
    qk_end = np.roll(qk, 3)  # element p: slot 5 of p - 3 is the end of QK(p)'s issue
    qk_end[:3] = np.nan
    print(f" QK issuer: issue call {med(qk_end - Kacq):.0f}; previous issue end -> buffer free {med(bfree[1:] - qk_end[:-1]):.0f};"
          f" buffer free -> K acquired {med(Kacq - bfree):.0f}; PV issuer saw element p-3 -> buffer free(p)"
          f" {med(bfree[3:] - seen0[:-3]):.0f}; K acquired -> S {med(S - Kacq):.0f}")
    if np.isfinite(mx).any():
        print(f" VSA frozen: S -> max taken {med(mx - S):.0f}; -> skip decided {med(dec - S):.0f}; -> consumed {med(P - S):.0f}")
    for i in range(20, min(26, n)):
        print(" ", np.round(tr[i, :15]).astype(int).tolist())
    sys.exit(0)
print(f"variant={a.variant} k_block={a.k_block} visited={n} total={np.nanmax(tr):.0f} cycles "
      f"-> {np.nanmax(tr) / n:.0f} cycles per block (both query tiles)")
for t in (0, 1):
    s_ready, p_done, p_seen, qk_iss = tr[:, 2 * t], tr[:, 2 * t + 1], tr[:, 4 + 2 * t], tr[:, 5 + 2 * t]
    busy = p_done - s_ready
    wait_s = s_ready[1:] - p_done[:-1]
    seen = p_seen - p_done
    qk_to_s = s_ready[1:] - qk_iss[:-1]
    sl = slice(4, n - 4)
    print(f" tile {t}: softmax busy median {np.nanmedian(busy[sl]):.0f} (p10 {np.nanpercentile(busy[sl], 10):.0f}"
          f" p90 {np.nanpercentile(busy[sl], 90):.0f}); softmax waits for S {np.nanmedian(wait_s[sl]):.0f};"
          f" MMA sees P after {np.nanmedian(seen[sl]):.0f}; S ready {np.nanmedian(qk_to_s[sl]):.0f} after QK issue;"
          f" period {np.nanmedian(np.diff(s_ready)[sl]):.0f}")
    if np.isfinite(tr[:, 18 + t]).any():  # warp-specialised kernel: first P chunk hand-off
        print(f"   tile {t}: first P chunk handed off {np.nanmedian((tr[:, 18 + t] - s_ready)[sl]):.0f} after S;"
              f" MMA sees it +{np.nanmedian((tr[:, 4 + 2 * t] - tr[:, 18 + t])[sl]):.0f};"
              f" last P chunk seen +{np.nanmedian((tr[:, 8 + 2 * t] - p_done)[sl]):.0f} after P done,"
              f" PV issued +{np.nanmedian((tr[:, 9 + 2 * t] - p_done)[sl]):.0f}")
print("blocks 20-25 (cycles rel. start): [sm0 S, sm0 P, sm1 S, sm1 P, mma0 P, mma0 QK, mma1 P, mma1 QK,"
      " mma0 lastP, mma0 PVdone, mma1 lastP, mma1 PVdone, K acq, sm0 enter, sm1 enter]")
for i in range(20, min(26, n)):
    print(" ", np.round(tr[i, :15]).astype(int).tolist())
print("producer / V: [V(g) TMA issued, K(g+1) TMA issued, MMA acquired V(g)]")
for i in range(20, min(26, n)):
    print(" ", np.round(tr[i, 15:18]).astype(int).tolist())
sl = slice(4, n - 4)
if np.isfinite(tr[:, 20]).any():  # warp-specialised kernel: MMA-side detail
    print(f" MMA: QK1 issued -> kv_empty commit done {np.nanmedian((tr[:, 20] - tr[:, 7])[sl]):.0f}; "
          f"-> V(g+1) acquired {np.nanmedian((tr[1:, 17] - tr[:-1, 20])[sl]):.0f}; "
          f"PV0 issued -> K acquired {np.nanmedian((tr[:, 12] - tr[:, 9])[sl]):.0f}; "
          f"K acquired -> QK0 issued {np.nanmedian((tr[:, 5] - tr[:, 12])[sl]):.0f}")
for t in (0, 1):
    if np.isfinite(tr[:, 21 + 4 * t]).any():  # warp-specialised kernel: inside one softmax block
        s0 = tr[:, 2 * t]
        print(f" tile {t} softmax: S loaded +{np.nanmedian((tr[:, 21 + 4 * t] - s0)[sl]):.0f}, chunk-0 P stored "
              f"+{np.nanmedian((tr[:, 22 + 4 * t] - s0)[sl]):.0f}, chunk-0 handed off +{np.nanmedian((tr[:, 18 + t] - s0)[sl]):.0f}, "
              f"chunk-1 handed off +{np.nanmedian((tr[:, 1 + 2 * t] - s0)[sl]):.0f}, row sum +{np.nanmedian((tr[:, 23 + 4 * t] - s0)[sl]):.0f}")
print(f" V TMA issue -> MMA acquires V: median {np.nanmedian((tr[:, 17] - tr[:, 15])[sl]):.0f}; "
      f"K(g+1) TMA issue -> K acquired (next block's slot 12): {np.nanmedian((tr[1:, 12] - tr[:-1, 16])[sl]):.0f}")
for t in (0, 1):
    sl = slice(4, n - 4)
    first, last, pvd, qk = tr[:, 4 + 2 * t], tr[:, 8 + 2 * t], tr[:, 9 + 2 * t], tr[:, 5 + 2 * t]
    print(f" tile {t}: MMA first->last P chunk {np.nanmedian((last - first)[sl]):.0f}; last P -> PV issued "
          f"{np.nanmedian((pvd - last)[sl]):.0f}; PV issued -> QK issued {np.nanmedian((qk - pvd)[sl]):.0f}")
    enter, sready, pdone_prev = tr[:, 13 + t], tr[:, 2 * t], np.roll(tr[:, 2 * t + 1], 1)
    print(f" tile {t}: softmax enters wait_s {np.nanmedian((enter - pdone_prev)[sl]):.0f} after its previous P; "
          f"waits {np.nanmedian((sready - enter)[sl]):.0f} in wait_s")
