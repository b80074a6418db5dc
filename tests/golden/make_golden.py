"""Generate golden vectors by running the REFERENCE package (vfa_lab) itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The output `tests/golden/golden.npz` is committed; nothing at test time reads
/root/reference. Inputs come from the reference's own generators
(src/tensor.py:92-181), rounded to bf16 (the kernels' input precision), and the
reference computes on the rounded values in float64.

Call-time hooks (no fork of the reference):
  * LSE capture: `finalize` is wrapped in vfa_lab.fa / vfa_lab.vfa / vfa_lab.sparse
    (imported by name at src/fa.py:13-22, src/vfa.py:23-34, src/sparse.py:17-28) to
    record m + log(l) per query block.
  * (n_sink, n_local): `build_schedule` is replaced in vfa_lab.vfa and vfa_lab.sparse
    by the generalisation of src/vfa.py:146-153 (identical at (1, 1)).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/reference/pkg/src")
import vfa_lab  # noqa: E402
import vfa_lab.fa as ref_fa  # noqa: E402
import vfa_lab.sparse as ref_sparse  # noqa: E402
import vfa_lab.vfa as ref_vfa  # noqa: E402
from vfa_lab import (AttentionProblem, BlockSpec, SkipConfig, gen_gaussian,  # noqa: E402
                     gen_structured)

HERE = os.path.dirname(os.path.abspath(__file__))


def bf16_round(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).to(torch.float64).numpy()


def bf16_bits(x):
    t = torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16)


_LSE = {}
_orig_finalize = ref_vfa.finalize


def _finalize_hook(state, row_base):
    with np.errstate(divide="ignore"):
        _LSE[row_base] = state.m + np.log(state.l)
    return _orig_finalize(state, row_base)


for mod in (ref_fa, ref_vfa, ref_sparse):
    mod.finalize = _finalize_hook

_orig_schedule = ref_vfa.build_schedule
_SCHED = {"n_sink": 1, "n_local": 1}


def _schedule_hook(i, vmax, local, reorder):
    ns, nl = _SCHED["n_sink"], _SCHED["n_local"]
    if (ns, nl) == (1, 1):
        return _orig_schedule(i, vmax, local, reorder)
    spec = sorted(j for j in (set(range(1, ns + 1)) | set(range(local - nl + 1, local + 1)))
                  if 1 <= j <= vmax)
    if not reorder:
        return ref_vfa.Schedule(tuple(range(1, vmax + 1)), frozenset(spec))
    tail = [j for j in range(1, vmax + 1) if j not in set(spec)]
    return ref_vfa.Schedule(tuple(spec + tail), frozenset(spec))


ref_vfa.build_schedule = _schedule_hook
ref_sparse.build_schedule = _schedule_hook


def run_case(name, spec, data, causal, variant, **kw):
    q, k, v = (bf16_round(x) for x in data)
    p = AttentionProblem(q=q, k=k, v=v, blocks=spec, causal=causal)
    _LSE.clear()
    _SCHED["n_sink"] = kw.pop("n_sink", 1)
    _SCHED["n_local"] = kw.pop("n_local", 1)
    rec = {"variant": variant, "causal": causal, "q_block": spec.q_block,
           "k_block": spec.k_block, "n_sink": _SCHED["n_sink"], "n_local": _SCHED["n_local"]}
    err = ""
    out = np.full(q.shape, np.nan)
    counters = stats = mon = trace = None
    try:
        if variant == "fa":
            out, counters, trace = vfa_lab.fa_forward(p)
        elif variant == "vfa":
            # monitor=True: the calibration gap is recorded too (src/vfa.py:217-221)
            out, counters, trace, mon = vfa_lab.vfa_forward(p, monitor=True, **kw)
        elif variant == "vsa":
            lam = kw.pop("lam")
            rec["lam"] = lam  # (recorded before the call: an error case keeps its parameters)
            out, counters, stats, mon = vfa_lab.vsa_forward(p, SkipConfig(lam=lam), monitor=True, **kw)
        elif variant == "blasst":
            lam, order = kw.pop("lam"), kw.pop("order", "sequential")
            rec["lam"], rec["order"] = lam, order
            out, counters, stats = vfa_lab.blasst_forward(p, SkipConfig(lam=lam), order=order)
        elif variant == "blasst_fa4":
            lam, tau = kw.pop("lam"), kw.pop("tau")
            rec["lam"], rec["tau"] = lam, tau
            out, counters, stats = vfa_lab.blasst_fa4_forward(p, SkipConfig(lam=lam, tau=tau))
        elif variant == "blasst_rowskip":
            lam = kw.pop("lam")
            rec["lam"] = lam
            out, counters, stats = vfa_lab.blasst_rowskip_forward(p, SkipConfig(lam=lam, granularity="row"))
        else:
            raise ValueError(variant)
    except (vfa_lab.FullyMaskedRowError, vfa_lab.NormalizerUnderflowError) as e:
        err = f"{type(e).__name__}:{e.row}"
    rec.update({k2: v2 for k2, v2 in kw.items()})
    lse = np.full(q.shape[0], np.nan)
    for base, val in _LSE.items():
        lse[base: base + spec.q_block] = val
    arrays = {}
    for t, x in (("q", q), ("k", k), ("v", v)):
        bits = bf16_bits(x)
        key = "in/" + hashlib.sha256(bits.tobytes()).hexdigest()[:16]
        arrays[key] = bits  # inputs shared by several cases are stored once
        rec[f"in_{t}"] = key
    arrays.update({
        # float32 copy for the GPU tolerance checks; the float64 result is pinned by
        # its sha256 (the oracle must reproduce it bit-for-bit)
        f"{name}/out": out.astype(np.float32), f"{name}/lse": lse,
    })
    if trace is not None:
        # StateTrace -> stabilization positions per row (src/analysis.py:39-78)
        rep = vfa_lab.stabilization_positions(trace)
        arrays[f"{name}/stab"] = rep.positions.astype(np.int32)
        rec["stab.frac_sink"], rec["stab.frac_local"], rec["stab.frac_other"] = (
            rep.frac_sink, rep.frac_local, rep.frac_other)
    rec["out_sha256"] = hashlib.sha256(np.ascontiguousarray(out, dtype=np.float64).tobytes()).hexdigest()
    if counters is not None:
        for f, val in counters.as_dict().items():
            rec[f"counters.{f}"] = val
    if stats is not None:
        for f in ("blocks_visited", "blocks_skipped", "processed_special", "processed_frozen",
                  "rescales_elided", "rows_masked", "row_slots", "blocks_processed"):
            rec[f"stats.{f}"] = getattr(stats, f)
    if mon is not None:
        rec["mon.count_over_f16"] = mon.count_over_f16
        rec["mon.count_over_f32"] = mon.count_over_f32
        rec["mon.exp_arg_max"] = mon.exp_arg_max
        if mon.calibration_gap is not None:
            for key, val in mon.calibration_gap.items():
                rec[f"mon.gap.{key}"] = val
    rec["error"] = err
    return arrays, rec


def main():
    cases = []
    # C1 exactly as BASELINE.json configs[0]: CPU oracle, block 64, 1 sink + 2 local.
    s = BlockSpec(1024, 1024, 64, 64, 64)
    cases.append(("c1_vfa_b64_s1l2", s, gen_gaussian(s, 0), True, "vfa", dict(n_local=2)))
    # C1 shape on the GPU tile geometry (Br=128, Bc=64): local band = 2 blocks.
    s = BlockSpec(1024, 1024, 64, 128, 64)
    cases.append(("c1_vfa_q128k64_s1l2", s, gen_gaussian(s, 1), True, "vfa", dict(n_local=2)))
    cases.append(("c1_fa_q128k64", s, gen_gaussian(s, 1), True, "fa", {}))
    s = BlockSpec(512, 512, 128, 128, 128)
    cases.append(("fa_d128_causal", s, gen_gaussian(s, 2), True, "fa", {}))
    cases.append(("vfa_d128_causal", s, gen_gaussian(s, 2), True, "vfa", {}))
    cases.append(("vfa_d128_causal_kmean", s, gen_gaussian(s, 3), True, "vfa", dict(kind="k_mean")))
    cases.append(("vfa_d128_noncausal_kmax_seq", s, gen_gaussian(s, 4), False, "vfa",
                  dict(kind="k_max", reorder=False)))
    cases.append(("vfa_d128_causal_noinit", s, gen_gaussian(s, 5), True, "vfa", dict(use_m_init=False)))
    cases.append(("vfa_d128_causal_tc1", s, gen_gaussian(s, 6), True, "vfa", dict(tc1=2)))
    # block-wise query representations for the m-init seed (src/vfa.py:69-76, 104-106)
    for qk in ("q_absmax", "q_sabsmax", "q_mean"):
        cases.append((f"vfa_d128_causal_{qk}", s, gen_gaussian(s, 14), True, "vfa", dict(qkind=qk)))
    cases.append(("vfa_d128_noncausal_q_sabsmax_kmax", s, gen_gaussian(s, 15), False, "vfa",
                  dict(qkind="q_sabsmax", kind="k_max")))
    s = BlockSpec(1024, 1024, 64, 128, 128)
    sd = gen_structured(s, 7, "middle_peak", 8.0)
    cases.append(("vsa_midpeak_lam1e-2", s, (sd.q, sd.k, sd.v), True, "vsa", dict(lam=1e-2)))
    cases.append(("vsa_midpeak_lam1e-9", s, (sd.q, sd.k, sd.v), True, "vsa", dict(lam=1e-9)))
    # planted sink (coordinate-0 trick of src/tensor.py:153-165, applied to block 1)
    q, k, v = gen_gaussian(s, 8)
    amp = np.sqrt(8.0 * np.sqrt(64))
    q[:, 0] = amp
    k[:, 0] = 0.0
    k[:128, 0] = amp
    cases.append(("vsa_sink_lam1e-2", s, (q, k, v), True, "vsa", dict(lam=1e-2)))
    sink = (q.copy(), k.copy(), v.copy())
    cases.append(("vsa_sink_lam1e-1", s, (q, k, v), True, "vsa", dict(lam=1e-1)))
    # frozen-max overflow without m-init (SURVEY.md §8d non-finite check)
    s = BlockSpec(512, 512, 128, 128, 128)
    sd = gen_structured(s, 9, "middle_peak", 120.0)
    cases.append(("vfa_overflow_noinit", s, (sd.q, sd.k, sd.v), True, "vfa", dict(use_m_init=False)))
    cases.append(("vfa_overflow_init", s, (sd.q, sd.k, sd.v), True, "vfa", dict(use_m_init=True)))
    # normalizer-underflow KAT (tests/test_cli.py:177-193) lifted to a 128x128 tile
    # (values scaled x5 so the seed gap exceeds float64's exp range at d=64, scale 1/8)
    q = np.zeros((128, 64)); q[:, :2] = 1.0
    k = np.zeros((128, 64)); k[0::2, 0], k[0::2, 1] = 6000.0, -6000.0
    k[1::2, 0], k[1::2, 1] = -6000.0, 6000.0
    v = np.ones((128, 64))
    s = BlockSpec(128, 128, 64, 128, 128)
    cases.append(("vfa_underflow_kmax", s, (q, k, v), False, "vfa", dict(kind="k_max")))

    # fp32 underflow window: k_absmax_unsigned seeds 100 nats above every score (q . k = 0 on
    # sign-balanced keys, q . |k| = 64 * 12.5 at scale 1/8). float64 normalizes (e^-100 is
    # representable); fp32 exp2 flushes to zero below e^-87.3, so the kernel must rebase
    q = np.ones((256, 64))
    k = np.full((256, 64), 12.5); k[:, 32:] = -12.5
    k[1::2] *= -1.0
    v = gen_gaussian(BlockSpec(256, 256, 64, 128, 128), 20)[2]
    s = BlockSpec(256, 256, 64, 128, 128)
    cases.append(("vfa_fp32_underflow_window", s, (q, k, v), True, "vfa", dict(kind="k_absmax_unsigned")))
    cases.append(("vsa_fp32_underflow_window", s, (q, k, v), True, "vsa", dict(kind="k_absmax_unsigned", lam=1e-3)))
    # beyond float64's range (seed 800 nats above every score): the reference raises too
    k2 = k * 8.0
    cases.append(("vfa_f64_underflow", s, (q, k2, v), True, "vfa", dict(kind="k_absmax_unsigned")))

    # BLASST family (src/sparse.py:112-253), SURVEY.md §8f row 1
    s = BlockSpec(1024, 1024, 64, 128, 128)
    mp = gen_structured(s, 11, "middle_peak", 8.0)
    mp = (mp.q, mp.k, mp.v)
    cases.append(("blasst_seq_sink_lam1e-2", s, sink, True, "blasst", dict(lam=1e-2)))
    cases.append(("blasst_swa_sink_lam1e-2", s, sink, True, "blasst", dict(lam=1e-2, order="sink_local")))
    cases.append(("blasst_nolam_gauss", s, gen_gaussian(s, 10), True, "blasst", dict(lam=None)))
    cases.append(("blasst_fa4_tau0_midpeak", s, mp, True, "blasst_fa4", dict(lam=None, tau=0.0)))
    cases.append(("blasst_fa4_tau8_sink_lam1e-3", s, sink, True, "blasst_fa4", dict(lam=1e-3, tau=8.0)))
    cases.append(("blasst_fa4_tauinf_gauss", s, gen_gaussian(s, 12), True, "blasst_fa4",
                  dict(lam=None, tau=float("inf"))))
    cases.append(("blasst_rowskip_sink_lam1e-3", s, sink, True, "blasst_rowskip", dict(lam=1e-3)))
    cases.append(("blasst_rowskip_nolam_gauss", s, gen_gaussian(s, 13), True, "blasst_rowskip", dict(lam=None)))
    s = BlockSpec(1024, 1024, 64, 128, 64)
    cases.append(("blasst_fa4_k64_tau2_sink", s, sink, True, "blasst_fa4", dict(lam=1e-2, tau=2.0)))
    cases.append(("blasst_rowskip_k64_midpeak_lam1e-2", s, mp, True, "blasst_rowskip", dict(lam=1e-2)))

    # query blocks smaller than the GPU's 128-row MMA tile (the reference CLI defaults to 64/64):
    # the GPU holds one reference block per tile, so schedules and statistics are the reference's
    s = BlockSpec(512, 512, 64, 64, 64)
    cases.append(("fa_q64k64_causal", s, gen_gaussian(s, 16), True, "fa", {}))
    cases.append(("vfa_q64k64_causal_s1l2", s, gen_gaussian(s, 17), True, "vfa", dict(n_local=2)))
    s = BlockSpec(512, 512, 128, 32, 64)
    cases.append(("vfa_q32k64_d128_causal", s, gen_gaussian(s, 18), True, "vfa", {}))
    s = BlockSpec(256, 256, 64, 16, 64)
    cases.append(("vfa_q16k64_noncausal_q_mean", s, gen_gaussian(s, 19), False, "vfa", dict(qkind="q_mean")))
    s = BlockSpec(1024, 1024, 64, 64, 128)
    cases.append(("vsa_sink_q64_lam1e-2", s, sink, True, "vsa", dict(lam=1e-2)))
    cases.append(("blasst_rowskip_sink_q64_lam1e-3", s, sink, True, "blasst_rowskip", dict(lam=1e-3)))
    s = BlockSpec(1024, 1024, 64, 32, 64)
    cases.append(("blasst_fa4_sink_q32_lam1e-3_tau8", s, sink, True, "blasst_fa4", dict(lam=1e-3, tau=8.0)))

    # head_dim 32 (the reference acceptance matrix runs d in {32, 64, 128}, tests/test_acceptance.py:37-61)
    # and 32-row key blocks
    s = BlockSpec(256, 256, 32, 64, 64)
    cases.append(("vfa_d32_q64k64_causal", s, gen_gaussian(s, 21), True, "vfa", {}))
    cases.append(("fa_d32_q64k64_noncausal", s, gen_gaussian(s, 22), False, "fa", {}))
    s = BlockSpec(512, 512, 32, 128, 128)
    cases.append(("vsa_d32_midpeak_lam1e-2", s, (lambda g: (g.q, g.k, g.v))(gen_structured(s, 23, "middle_peak", 8.0)),
                  True, "vsa", dict(lam=1e-2)))
    s = BlockSpec(512, 512, 128, 128, 32)
    cases.append(("vfa_k32_d128_causal", s, gen_gaussian(s, 24), True, "vfa", {}))
    cases.append(("fa_k32_d128_causal", s, gen_gaussian(s, 24), True, "fa", {}))
    s = BlockSpec(512, 512, 64, 64, 32)
    cases.append(("vfa_k32_d64_q64_noncausal_kmax", s, gen_gaussian(s, 25), False, "vfa", dict(kind="k_max")))
    s = BlockSpec(1024, 1024, 64, 128, 32)
    cases.append(("blasst_fa4_k32_sink_lam1e-3_tau2", s, sink, True, "blasst_fa4", dict(lam=1e-3, tau=2.0)))

    arrays, meta = {}, []
    for name, spec, data, causal, variant, kw in cases:
        a, rec = run_case(name, spec, data, causal, variant, **dict(kw))
        rec["name"] = name
        arrays.update(a)
        meta.append(rec)
        print(name, {k2: v2 for k2, v2 in rec.items() if k2.startswith(("stats", "error", "mon.count"))})
    arrays["meta"] = np.array(json.dumps(meta))  # json: carries inf / nan (tau = inf)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)


if __name__ == "__main__":
    main()
