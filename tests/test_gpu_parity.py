"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Inputs are bf16; the oracle computes in float64 on the identical (upcast) values.
Tolerances (bf16 inputs, fp32 S / l / O accumulation, bf16 P and bf16 O):
  O   : max |O_gpu - O_ref| <= 2e-2 (one bf16 ulp of |O| in [2, 4)) and
        max_rel_err (tests/conftest.py:42-46 metric) <= 1e-2
  LSE : max |LSE_gpu - LSE_ref| <= 1e-4
  visit statistics (visited / special / frozen / skipped): exact
  VSA skip decisions: exact wherever the oracle's decision margin exceeds 1e-3
  OverflowMonitor counts: equal up to the arguments within 5e-3 of a threshold; exp_arg_max and
  the calibration gap within 1e-2 (fp32 scores against float64)
"""

import zlib

import numpy as np
import pytest
import torch

from golden_io import case, case_bits, case_names, case_stab
from oracle import vfa_oracle as vo

pytestmark = pytest.mark.gpu

O_ABS, O_REL, LSE_ABS = 2e-2, 1e-2, 1e-4
MON_TOL = 1e-2


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2604_12798_b200 import build
    build.build()


def _rand(shape, seed, dev="cuda"):
    g = torch.Generator(device=dev).manual_seed(seed)
    return torch.randn(shape, generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)


def _f64(t):
    return t.float().cpu().numpy().astype(np.float64)


def _run_gpu(q, k, v, **kw):
    from paper_2604_12798_b200 import attention_forward, stats_dict
    out, lse, info = attention_forward(q, k, v, check=False, **kw)
    torch.cuda.synchronize()
    return out, lse, info, stats_dict(info)


def _compare(out, lse, ref_o, ref_lse, tag=""):
    o = _f64(out)
    l = lse.double().cpu().numpy()
    assert np.isfinite(o).all(), f"{tag}: non-finite output"
    err = np.abs(o - ref_o).max()
    rel = vo.max_rel_err(o, ref_o)
    lerr = np.abs(l - ref_lse).max()
    assert err <= O_ABS, f"{tag}: O max abs err {err}"
    assert rel <= O_REL, f"{tag}: O max_rel_err {rel}"
    assert lerr <= LSE_ABS, f"{tag}: LSE max abs err {lerr}"
    return err, rel, lerr


CONFIGS = []
for variant in ("fa", "vfa", "vsa"):
    for d in (64, 128):
        for bc in (64, 128):
            for causal in (True, False):
                CONFIGS.append((variant, d, bc, causal))


@pytest.mark.parametrize("variant,d,bc,causal", CONFIGS)
def test_parity_matrix(variant, d, bc, causal):
    B, Hq, Hkv, L = 1, 2, 1, 512
    seed = zlib.crc32(repr((variant, d, bc, causal)).encode()) % 1000  # reproducible across runs
    q, k, v = _rand((B, Hq, L, d), seed), _rand((B, Hkv, L, d), seed + 1), _rand((B, Hkv, L, d), seed + 2)
    kw = dict(variant=variant, causal=causal, q_block=128, k_block=bc)
    if variant == "vsa":
        kw["lam"] = 1e-2
    out, lse, info, st = _run_gpu(q, k, v, **kw)
    ref_o, ref_lse, ref_st = vo.forward(_f64(q), _f64(k), _f64(v), **kw)
    _compare(out, lse, ref_o, ref_lse, str(kw))
    for key in ("visited", "special", "frozen"):
        if variant != "vsa":
            assert st[key] == ref_st[key], (key, st, ref_st)
    assert st["visited"] == ref_st["visited"]


@pytest.mark.parametrize("hq,hkv,b", [(1, 1, 1), (3, 1, 1), (8, 2, 2), (4, 4, 1)])
def test_gqa_and_single_tile_paths(hq, hkv, b):
    L, d = 384, 128
    q, k, v = _rand((b, hq, L, d), 11), _rand((b, hkv, L, d), 12), _rand((b, hkv, L, d), 13)
    for variant in ("fa", "vfa"):
        kw = dict(variant=variant, causal=True, q_block=128, k_block=128)
        out, lse, _, st = _run_gpu(q, k, v, **kw)
        ref_o, ref_lse, ref_st = vo.forward(_f64(q), _f64(k), _f64(v), **kw)
        _compare(out, lse, ref_o, ref_lse, f"{variant} hq={hq} hkv={hkv} b={b}")
        assert (st["special"], st["frozen"]) == (ref_st["special"], ref_st["frozen"])


@pytest.mark.parametrize("kind", ["sabsmax", "k_max", "k_mean", "k_absmax_unsigned"])
@pytest.mark.parametrize("opts", [dict(), dict(reorder=False), dict(use_m_init=False), dict(tc1=2),
                                  dict(n_sink=2, n_local=2), dict(n_sink=1, n_local=2, k_block=64),
                                  dict(n_sink=0, n_local=1)])
def test_vfa_options(kind, opts):
    L, d = 640, 128
    q, k, v = _rand((1, 2, L, d), 21), _rand((1, 1, L, d), 22), _rand((1, 1, L, d), 23)
    kw = dict(variant="vfa", causal=True, q_block=128, k_block=128, kind=kind)
    kw.update(opts)
    out, lse, _, st = _run_gpu(q, k, v, **kw)
    ref_o, ref_lse, ref_st = vo.forward(_f64(q), _f64(k), _f64(v), **kw)
    _compare(out, lse, ref_o, ref_lse, str(kw))
    assert (st["special"], st["frozen"]) == (ref_st["special"], ref_st["frozen"])


def _golden_kw(m):
    kw = dict(variant=m["variant"], causal=m["causal"], q_block=m["q_block"], k_block=m["k_block"],
              n_sink=m["n_sink"], n_local=m["n_local"])
    for key in ("kind", "qkind", "reorder", "use_m_init", "tc1", "lam", "tau"):
        if key in m:
            kw[key] = m[key]
    if m.get("order") == "sink_local":
        kw["reorder"] = True
    return kw


@pytest.mark.parametrize("name", [n for n in case_names()])
def test_golden_vectors(name):
    m, q, k, v, out32, lse = case(name)
    from paper_2604_12798_b200 import attention_forward, stats_dict
    from paper_2604_12798_b200.api import NormalizerUnderflowError
    qb, kb, vb = (torch.from_numpy(x.astype(np.int16)).view(torch.bfloat16).cuda()[None, None]
                  for x in case_bits(name))
    kw = _golden_kw(m)
    if m["error"]:
        with pytest.raises(NormalizerUnderflowError) as ei:
            attention_forward(qb, kb, vb, **kw)
        assert ei.value.row == int(m["error"].split(":")[1])
        return
    # check=True: the fp32 underflow window rows are rebased (vfa_fwd_rebased) like the reference
    out, lse_g, info = attention_forward(qb, kb, vb, check=True, monitor=True, **kw)
    st = stats_dict(info)
    if m.get("mon.count_over_f32", 0) > 0:
        # frozen-max overflow: float64 stays finite, fp32 exp2 may not; must be reported
        assert st["count_over_f32"] > 0
        o = _f64(out[0, 0])
        if not np.isfinite(o).all():
            assert st["nonfinite_rows"] > 0
        return
    _compare(out[0, 0], lse_g[0, 0], out32.astype(np.float64), lse, name)
    if "mon.count_over_f32" in m and not info.get("rebased_rows"):
        _check_monitor(st, m, q, k, v, kw)
    stab = case_stab(name)
    if stab is not None:
        # device StateTrace stabilization positions vs the reference's (fp32 vs float64 maxima:
        # a row whose two largest block maxima tie within fp32 rounding may differ)
        _, _, info2 = attention_forward(qb, kb, vb, check=False, stab_trace=True, **kw)
        got = info2["stab_block"][0, 0].cpu().numpy()
        assert (got != stab).mean() <= 0.01, (name, (got != stab).sum())
    if "stats.blocks_visited" in m:
        assert st["visited"] == m["stats.blocks_visited"]
        assert st["skipped"] == m["stats.blocks_skipped"]
        if m["variant"] == "vsa":
            assert st["special"] == m["stats.processed_special"]
            assert st["frozen"] == m["stats.processed_frozen"]
        if "stats.blocks_processed" in m:
            assert st["special"] + st["frozen"] == m["stats.blocks_processed"]
            assert st["elided"] == m["stats.rescales_elided"]
            assert st["rows_masked"] == m["stats.rows_masked"]
    if "counters.rescale_events" in m and m["variant"] in ("fa", "vfa"):
        assert st["special"] == m["counters.rescale_events"]
        assert st["special"] + st["frozen"] == m["counters.blocks_processed"]


def _check_monitor(st, m, q, k, v, kw):
    """OverflowMonitor on the device vs the reference (src/vfa.py:109-135)."""
    r = vo.forward_head(q, k, v, monitor=True, raise_errors=False,
                        **{key: val for key, val in kw.items() if key not in ("variant",)}, variant=kw["variant"])
    for lim in ("f16", "f32"):
        ref = m[f"mon.count_over_{lim}"]
        near = getattr(r.monitor, f"near_{lim}")
        assert abs(st[f"count_over_{lim}"] - ref) <= near, (lim, st[f"count_over_{lim}"], ref, near)
    assert abs(st["exp_arg_max"] - m["mon.exp_arg_max"]) <= MON_TOL * max(1.0, abs(m["mon.exp_arg_max"]))
    if "mon.gap.min" in m:
        g = st["calibration_gap"]
        assert g is not None
        for key in ("min", "max", "mean"):
            assert abs(g[key] - m[f"mon.gap.{key}"]) <= MON_TOL, (key, g[key], m[f"mon.gap.{key}"])
        # rows whose seed equals the exact max within fp32 rounding may fall on either side of 0
        amb = float((np.abs(r.monitor.gap) <= 1e-3).mean())
        assert abs(g["frac_below"] - m["mon.gap.frac_below"]) <= amb + 1e-12
    else:
        assert st["calibration_gap"] is None


@pytest.mark.parametrize("name", [n for n in case_names() if n.startswith("blasst")])
def test_blasst_golden_counters_integer_equal(name):
    # the reference-shaped entry points charge OpCounters from the device's block-class
    # counts: integer-equal to the reference's instrumented counters (src/counters.py)
    from paper_2604_12798_b200 import (AttentionProblem, BlockSpec, SkipConfig, blasst_fa4_forward,
                                       blasst_forward, blasst_rowskip_forward)
    m, q, k, v, out32, lse = case(name)
    qb, kb, vb = (torch.from_numpy(x.astype(np.int16)).view(torch.bfloat16).cuda() for x in case_bits(name))
    L, d = qb.shape
    p = AttentionProblem(qb, kb, vb, blocks=BlockSpec(L, L, d, m["q_block"], m["k_block"]), causal=m["causal"])
    if m["variant"] == "blasst":
        out, c, stats = blasst_forward(p, SkipConfig(lam=m["lam"]), order=m.get("order", "sequential"))
    elif m["variant"] == "blasst_fa4":
        out, c, stats = blasst_fa4_forward(p, SkipConfig(lam=m["lam"], tau=m["tau"]))
    else:
        out, c, stats = blasst_rowskip_forward(p, SkipConfig(lam=m["lam"], granularity="row"))
    for f, val in c.as_dict().items():
        assert val == m[f"counters.{f}"], (f, val, m[f"counters.{f}"])
    for f in ("blocks_visited", "blocks_skipped", "rescales_elided", "rows_masked", "row_slots",
              "blocks_processed"):
        assert getattr(stats, f) == m[f"stats.{f}"], f
    assert vo.max_rel_err(_f64(out), out32.astype(np.float64)) <= O_REL


BLASST_CASES = [("blasst", dict(lam=1e-2)), ("blasst", dict(lam=1e-2, reorder=True)),
                ("blasst", dict(lam=None)), ("blasst_fa4", dict(lam=None, tau=0.0)),
                ("blasst_fa4", dict(lam=1e-3, tau=8.0)), ("blasst_fa4", dict(lam=None, tau=float("inf"))),
                ("blasst_rowskip", dict(lam=1e-3)), ("blasst_rowskip", dict(lam=None))]


@pytest.mark.parametrize("variant,opts", BLASST_CASES)
@pytest.mark.parametrize("d,bc", [(128, 128), (64, 64)])
def test_blasst_family_against_oracle(variant, opts, d, bc):
    # planted sink (src/tensor.py:153-165 trick) so that skips / elisions / masked rows occur
    B, Hq, Hkv, L = 1, 4, 2, 1024
    q, k, v = _rand((B, Hq, L, d), 121), _rand((B, Hkv, L, d), 122), _rand((B, Hkv, L, d), 123)
    amp = float(np.sqrt(8.0 * np.sqrt(d)))
    q[..., 0] = amp
    k[..., 0] = 0
    k[:, :, :bc, 0] = amp
    kw = dict(variant=variant, causal=True, q_block=128, k_block=bc, **opts)
    order = "sink_local" if opts.get("reorder") else "sequential"
    okw = {key: val for key, val in kw.items() if key != "reorder"}
    out, lse, _, st = _run_gpu(q, k, v, **kw)
    qf, kf, vf = _f64(q), _f64(k), _f64(v)
    o_ref = np.empty(out.shape)
    l_ref = np.empty(lse.shape)
    ref = {"visited": 0, "skipped": 0, "elided": 0, "rows_masked": 0}
    tight = True
    for h in range(Hq):
        r = vo.forward_head(qf[0, h], kf[0, h // 2], vf[0, h // 2], order=order, record_decisions=True, **okw)
        o_ref[0, h], l_ref[0, h] = r.out, r.lse
        for key in ref:
            ref[key] += getattr(r, key)
        tight &= all(mg > 1e-3 for blk in r.decisions for (_, _, mg) in blk)
    _compare(out, lse, o_ref, l_ref, str(kw))
    assert st["visited"] == ref["visited"]
    if tight:  # no decision within fp32 rounding of its threshold: counts are exact
        assert st["skipped"] == ref["skipped"]
        assert st["rows_masked"] == ref["rows_masked"]
    if variant != "blasst_fa4" or opts["tau"] in (float("inf"),):
        assert st["elided"] == ref["elided"]


@pytest.mark.parametrize("split", [2, 4])
def test_blasst_without_threshold_is_bitwise_fa(split):
    # reference tests/test_sparse.py:32-38 (blasst) and :122-128 (rowskip): lam=None -> FA
    q, k, v = _rand((1, 4, 1024, 128), 131), _rand((1, 2, 1024, 128), 132), _rand((1, 2, 1024, 128), 133)
    base = dict(causal=True, softmax_split=split)
    o_fa, l_fa, _, _ = _run_gpu(q, k, v, variant="fa", **base)
    for variant in ("blasst", "blasst_rowskip"):
        o, l, _, st = _run_gpu(q, k, v, variant=variant, lam=None, reorder=False, **base)
        assert st["skipped"] == 0 and st["rows_masked"] == 0
        assert torch.equal(o, o_fa) and torch.equal(l, l_fa), variant


def test_blasst_fa4_tau_zero_equals_plain_skip():
    # reference tests/test_sparse.py:184-192: tau = 0 elides only where the max did not rise,
    # which changes nothing numerically
    q, k, v = _rand((1, 4, 1024, 128), 141), _rand((1, 2, 1024, 128), 142), _rand((1, 2, 1024, 128), 143)
    o1, l1, _, s1 = _run_gpu(q, k, v, variant="blasst", lam=1e-3, causal=True, reorder=False)
    o2, l2, _, s2 = _run_gpu(q, k, v, variant="blasst_fa4", lam=1e-3, tau=0.0, causal=True)
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    assert s1["skipped"] == s2["skipped"]


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("bc", [64, 128])
@pytest.mark.parametrize("kind", ["sabsmax", "k_max", "k_mean", "k_absmax_unsigned"])
def test_krepr_kernel(d, bc, kind):
    from paper_2604_12798_b200 import AttentionProblem, BlockSpec, precompute_kreprs
    L = 1024
    k = _rand((2, 3, L, d), 31)
    k[0, 0, 5, 3] = -k[0, 0, 7, 3].abs() - 1  # planted ties / signs
    q = _rand((2, 3, L, d), 32)
    p = AttentionProblem(q, k, k, blocks=BlockSpec(L, L, d, 128, bc))
    got = _f64(precompute_kreprs(p, kind))
    kk = _f64(k)
    for b in range(2):
        for h in range(3):
            ref = np.stack(vo.precompute_kreprs(kk[b, h], bc, kind))
            if kind == "k_mean":
                assert np.abs(got[b, h] - ref).max() <= 2e-2 * np.abs(ref).max() + 1e-3
            else:
                assert np.array_equal(got[b, h], ref)  # selected elements: exact in bf16


def _planted_sink(L, d, boost, seed, hq=2):
    q, k, v = _rand((1, hq, L, d), seed), _rand((1, 1, L, d), seed + 1), _rand((1, 1, L, d), seed + 2)
    amp = float(np.sqrt(boost * np.sqrt(d)))
    q[..., 0] = amp
    k[..., 0] = 0
    k[:, :, :128, 0] = amp
    return q, k, v


@pytest.mark.parametrize("lam", [1e-4, 1e-3, 3e-3, 1e-2, 1e-1])
def test_vsa_skip_decisions(lam):
    L, d = 2048, 128
    q, k, v = _planted_sink(L, d, 8.0, 41)
    kw = dict(variant="vsa", causal=True, q_block=128, k_block=128, lam=lam)
    from paper_2604_12798_b200 import attention_forward
    out, lse, info = attention_forward(q, k, v, check=False, skip_trace=True, **kw)
    trace = info["skip_trace"].cpu().numpy()
    qq, kk, vv = _f64(q), _f64(k), _f64(v)
    ref_o = np.empty(qq.shape)
    flips = 0
    for h in range(2):
        r = vo.forward_head(qq[0, h], kk[0, 0], vv[0, 0], record_decisions=True, **kw)
        ref_o[0, h] = r.out
        for i, dec in enumerate(r.decisions):
            for pos, (j, skip, margin) in enumerate(dec):
                g = trace[0, h, i, pos]
                assert g in (1, 2)
                if margin > 1e-3:
                    assert (g == 2) == skip, (h, i, pos, j, margin)
                elif (g == 2) != skip:
                    flips += 1
    assert flips <= 2
    if flips == 0:
        assert np.abs(_f64(out) - ref_o).max() <= O_ABS


@pytest.mark.parametrize("split", [2, 4])
def test_vsa_tiny_lambda_bitwise_equals_vfa(split):
    # reference tests/test_sparse.py:148-153 on the device path (same softmax layout)
    q, k, v = _rand((1, 4, 1024, 128), 51), _rand((1, 2, 1024, 128), 52), _rand((1, 2, 1024, 128), 53)
    base = dict(causal=True, q_block=128, k_block=128, softmax_split=split)
    o1, l1, _, _ = _run_gpu(q, k, v, variant="vfa", **base)
    o2, l2, _, st = _run_gpu(q, k, v, variant="vsa", lam=1e-9, **base)
    assert st["skipped"] == 0
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


@pytest.mark.parametrize("split", [2, 4])
def test_single_key_block_vfa_equals_fa(split):
    # reference tests/test_vfa.py:115-125: T_c = 1 -> the one block is special
    q, k, v = _rand((1, 2, 128, 64), 61), _rand((1, 1, 128, 64), 62), _rand((1, 1, 128, 64), 63)
    o1, l1, _, _ = _run_gpu(q, k, v, variant="fa", causal=True, softmax_split=split)
    o2, l2, _, _ = _run_gpu(q, k, v, variant="vfa", causal=True, use_m_init=False, softmax_split=split)
    assert torch.equal(o1, o2) and torch.equal(l1, l2)


@pytest.mark.parametrize("variant", ["fa", "vfa", "vsa"])
@pytest.mark.parametrize("d,bc", [(128, 128), (64, 64), (128, 64), (64, 128)])
def test_softmax_splits_agree_with_oracle(variant, d, bc):
    # every softmax layout (1, 2 or 4 threads per row) against the oracle, and the per-variant
    # default is one of them
    B, Hq, Hkv, L = 1, 4, 2, 512
    q, k, v = _rand((B, Hq, L, d), 111), _rand((B, Hkv, L, d), 112), _rand((B, Hkv, L, d), 113)
    kw = dict(variant=variant, causal=True, q_block=128, k_block=bc)
    if variant == "vsa":
        kw["lam"] = 1e-2
    ref_o, ref_lse, ref_st = vo.forward(_f64(q), _f64(k), _f64(v), **kw)
    outs = {}
    for split in (0, 1, 2, 4):
        out, lse, _, st = _run_gpu(q, k, v, softmax_split=split, **kw)
        _compare(out, lse, ref_o, ref_lse, f"{kw} split={split}")
        assert st["visited"] == ref_st["visited"]
        outs[split] = out
    # the default (0) runs the warp-specialised kernel at d = Bc = 128 (its own layout, checked
    # against the oracle above), and one of the explicit layouts elsewhere
    if (d, bc) != (128, 128):
        assert any(torch.equal(outs[0], outs[sp]) for sp in (1, 2, 4))


def test_deterministic_and_head_sharding_invariant():
    q, k, v = _rand((1, 8, 1024, 128), 71), _rand((1, 2, 1024, 128), 72), _rand((1, 2, 1024, 128), 73)
    o1, l1, _, _ = _run_gpu(q, k, v, variant="vfa", causal=True)
    o2, l2, _, _ = _run_gpu(q, k, v, variant="vfa", causal=True)
    assert torch.equal(o1, o2)
    # shard by KV-head group exactly as bench.py does for multi-GPU runs
    o3, l3, _, _ = _run_gpu(q[:, 4:].contiguous(), k[:, 1:].contiguous(), v[:, 1:].contiguous(),
                            variant="vfa", causal=True)
    assert torch.equal(o1[:, 4:], o3) and torch.equal(l1[:, 4:], l3)


def test_strided_inputs():
    base = _rand((1, 1024, 4, 128), 81)  # [B, L, H, d] layout viewed as [B, H, L, d]
    q = base.permute(0, 2, 1, 3)
    kv = _rand((1, 1024, 2, 128), 82).permute(0, 2, 1, 3)
    out, lse, _, _ = _run_gpu(q, kv, kv, variant="vfa", causal=True)
    ref_o, ref_lse, _ = vo.forward(_f64(q), _f64(kv), _f64(kv), variant="vfa", causal=True,
                                   q_block=128, k_block=128)
    _compare(out, lse, ref_o, ref_lse, "strided")


def test_large_context_sampled_head():
    # C2 geometry per head (d=128, Bc=128) at L=8192: one head checked against the oracle
    L = 8192
    q, k, v = _rand((1, 4, L, 128), 91), _rand((1, 1, L, 128), 92), _rand((1, 1, L, 128), 93)
    out, lse, _, st = _run_gpu(q, k, v, variant="vfa", causal=True)
    r = vo.forward_head(_f64(q[0, 3]), _f64(k[0, 0]), _f64(v[0, 0]), variant="vfa", causal=True,
                        q_block=128, k_block=128)
    _compare(out[0, 3], lse[0, 3], r.out, r.lse, "L=8192")
    t_r = L // 128
    assert st["special"] == 4 * sum(min(2, i) for i in range(1, t_r + 1))


def test_validation_errors_raise_like_reference():
    from paper_2604_12798_b200 import attention_forward
    q = _rand((1, 1, 200, 128), 1)
    with pytest.raises(ValueError):
        attention_forward(q, q, q, variant="vfa")  # 200 % 128 != 0 (src/tensor.py:37-44)
    q = _rand((1, 1, 256, 128), 1)
    with pytest.raises(ValueError):
        attention_forward(q, q, q, variant="vsa", lam=1.5)
    with pytest.raises(ValueError):
        attention_forward(q, q, q, variant="vfa", kind="median")
    with pytest.raises(ValueError):
        attention_forward(q, q, q, variant="vfa", q_block=48)
    k = _rand((1, 1, 128, 128), 2)
    with pytest.raises(ValueError):
        attention_forward(q, k, k, variant="fa", causal=True)  # causal needs Nq == Nk


def test_dropin_api_mirrors_reference():
    # reference-shaped call: 2-D single head, numpy inputs, tuple results
    from paper_2604_12798_b200 import (AttentionProblem, BlockSpec, SkipConfig, fa_forward,
                                       vfa_forward, vsa_forward)
    rng = np.random.default_rng(5)
    L, d = 512, 64
    q, k, v = (torch.from_numpy(rng.normal(size=(L, d))).to(torch.bfloat16) for _ in range(3))
    qf, kf, vf = (x.double().numpy() for x in (q, k, v))
    p = AttentionProblem(q, k, v, blocks=BlockSpec(L, L, d, 128, 128), causal=True)
    out, counters, trace, mon = vfa_forward(p)
    r = vo.forward_head(qf, kf, vf, variant="vfa", causal=True, q_block=128, k_block=128)
    from paper_2604_12798_b200 import DeviceTrace
    assert out.shape == (L, d) and isinstance(trace, DeviceTrace)
    assert np.array_equal(trace.positions.cpu().numpy(), r.stab) or (trace.positions.cpu().numpy() != r.stab).mean() < 0.01
    assert vo.max_rel_err(_f64(out), r.out) <= O_REL
    t_r = L // 128
    assert counters.rowmax_reductions == sum(min(2, i) for i in range(1, t_r + 1))
    assert counters.blocks_processed == sum(range(1, t_r + 1))
    o2, c2, _ = fa_forward(p)
    assert c2.rescale_events == sum(range(1, t_r + 1))
    o3, c3, stats, _ = vsa_forward(p, SkipConfig(lam=1e-9))
    assert stats.blocks_skipped == 0 and torch.equal(o3, out)
    assert c3.rowmax_reductions == stats.blocks_visited


@pytest.mark.parametrize("variant,chunk,qchunk,b", [("vfa", 1, 2, 1), ("fa", 2, 0, 1), ("vsa", 1, 1, 2),
                                                     ("vfa", 4, 0, 2), ("blasst_fa4", 1, 0, 1)])
def test_host_pipeline_bitwise_equals_device_path(variant, chunk, qchunk, b):
    # vfa_fwd_host (chunked H2D / kernels / D2H) computes exactly what vfa_fwd computes
    from paper_2604_12798_b200 import attention_forward, stats_dict
    L, Hq, Hkv = 1024, 8, 4
    q, k, v = _rand((b, Hq, L, 128), 101), _rand((b, Hkv, L, 128), 102), _rand((b, Hkv, L, 128), 103)
    kw = dict(variant=variant, causal=True, lam=1e-2 if variant != "vfa" else None)
    if qchunk == 1:  # one query head per kernel launch runs the 4-way softmax split: match it
        kw["softmax_split"] = 4
    if variant == "blasst_fa4":
        kw["tau"] = 2.0
    o1, l1, i1, st1 = _run_gpu(q, k, v, **kw)
    qh, kh, vh = (x.cpu().pin_memory() for x in (q, k, v))
    from paper_2604_12798_b200 import attention_forward_host
    o2, l2, i2 = attention_forward_host(qh, kh, vh, chunk_kv_heads=chunk, chunk_q_heads=qchunk, **kw)
    assert o2.device.type == "cpu" and l2.device.type == "cpu"
    assert torch.equal(o1.cpu(), o2) and torch.equal(l1.cpu(), l2)
    assert stats_dict(i2) == st1
    # and through the generic entry point with CPU tensors (pageable memory works too)
    o3, l3, _ = attention_forward(q.cpu(), k.cpu(), v.cpu(), **kw)
    assert torch.equal(o3, o2) and torch.equal(l3, l2)


@pytest.mark.parametrize("variant", ["vfa", "vsa", "fa"])
def test_long_rows_host_pipeline_and_reruns_bitwise(variant):
    # long rows (128 key blocks per query tile at the end) through the warp-specialised kernels:
    # reruns and the host pipeline (kernels on two overlapping streams) are bitwise equal to the
    # device path -- a cross-thread TMEM hazard between the two halves of an S row (P of one half
    # stored over S columns the other half was still loading) showed up only this way
    from paper_2604_12798_b200 import attention_forward
    L, Hq, Hkv = 16384, 4, 1
    q, k, v = _rand((1, Hq, L, 128), 201), _rand((1, Hkv, L, 128), 202), _rand((1, Hkv, L, 128), 203)
    kw = dict(variant=variant, causal=True, lam=1e-2 if variant == "vsa" else None)
    o1, l1, _, _ = _run_gpu(q, k, v, **kw)
    o2, l2, _, _ = _run_gpu(q, k, v, **kw)
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    qh, kh, vh = (x.cpu().pin_memory() for x in (q, k, v))
    o3, l3, _ = attention_forward(qh, kh, vh, **kw)
    assert torch.equal(o3, o1.cpu()) and torch.equal(l3, l1.cpu())


@pytest.mark.parametrize("qkind", ["q_absmax", "q_mean", "q_sabsmax"])
@pytest.mark.parametrize("variant", ["vfa", "vsa"])
def test_host_pipeline_blockwise_qkind_gqa4(qkind, variant):
    # block-wise query representations through the chunked host pipeline with GQA group 4 and
    # query sub-chunks of 2 heads: every sub-chunk has its own seed area (sub-chunks of one K/V
    # group run on alternating streams), so the result equals the device path bitwise
    from paper_2604_12798_b200 import attention_forward_host
    L, Hq, Hkv = 1024, 8, 2
    q, k, v = _rand((1, Hq, L, 128), 111), _rand((1, Hkv, L, 128), 112), _rand((1, Hkv, L, 128), 113)
    # (lam=None: the block-wise seeds are loose upper bounds, at lambda 1e-2 every block of some
    # rows would be skipped -- a NormalizerUnderflowError in the reference as well)
    kw = dict(variant=variant, causal=True, qkind=qkind, lam=None)
    o1, l1, _, st1 = _run_gpu(q, k, v, **kw)
    qh, kh, vh = (x.cpu().pin_memory() for x in (q, k, v))
    for _ in range(3):  # races would show up as run-to-run differences
        o2, l2, i2 = attention_forward_host(qh, kh, vh, chunk_kv_heads=1, chunk_q_heads=2, **kw)
        assert torch.equal(o1.cpu(), o2) and torch.equal(l1.cpu(), l2)
    ref_o, ref_lse, _ = vo.forward(_f64(q), _f64(k), _f64(v), q_block=128, k_block=128, **kw)
    _compare(o1, l1, ref_o, ref_lse, f"{variant} {qkind}")


def test_host_pipeline_reports_whole_problem_row():
    # the golden normalizer-underflow case (reference tests/test_cli.py:177-193 geometry at
    # Br=Bc=128) placed at (batch 1, head 1) of a 2x2-head problem that runs as 4 chunks: the
    # status must carry the whole-problem linear row ((b * Hq + h) * L + r)
    from paper_2604_12798_b200 import attention_forward_host
    from paper_2604_12798_b200.api import NormalizerUnderflowError
    name = "vfa_underflow_kmax"
    m = case(name)[0]
    qb, kb, vb = (torch.from_numpy(x.astype(np.int16)).view(torch.bfloat16) for x in case_bits(name))
    B, H, (L, d) = 2, 2, qb.shape
    q, k, v = (_rand((B, H, L, d), 7 + i, dev="cpu") for i in range(3))
    q[1, 1], k[1, 1], v[1, 1] = qb, kb, vb
    with pytest.raises(NormalizerUnderflowError) as ei:
        attention_forward_host(q, k, v, variant="vfa", kind=m["kind"], causal=m["causal"],
                               k_block=m["k_block"], chunk_kv_heads=1, chunk_q_heads=1)
    assert ei.value.row == (1 * H + 1) * L + int(m["error"].split(":")[1])


def test_device_trace_stabilization_api():
    # reference-shaped: fa_forward returns a trace that stabilization_positions consumes
    # (tests/test_acceptance.py:171-183 pattern, on the golden planted-middle-peak problem)
    from paper_2604_12798_b200 import (AttentionProblem, BlockSpec, fa_forward, stabilization_positions,
                                       vfa_forward)
    name = "vsa_midpeak_lam1e-2"
    m, q, k, v, _, _ = case(name)
    qb, kb, vb = (torch.from_numpy(x.astype(np.int16)).view(torch.bfloat16).cuda() for x in case_bits(name))
    L, d = qb.shape
    p = AttentionProblem(qb, kb, vb, blocks=BlockSpec(L, L, d, 128, m["k_block"]), causal=True)
    _, _, trace = fa_forward(p)
    rep = stabilization_positions(trace)
    r = vo.forward_head(q, k, v, variant="fa", causal=True, q_block=128, k_block=m["k_block"])
    assert (rep.positions != r.stab).mean() <= 0.01
    assert abs(rep.frac_sink + rep.frac_local + rep.frac_other - 1.0) < 1e-12
    _, _, vtrace, _ = vfa_forward(p)
    rv = vo.forward_head(q, k, v, variant="vfa", causal=True, q_block=128, k_block=m["k_block"])
    assert (vtrace.positions.cpu().numpy() != rv.stab).mean() <= 0.01


@pytest.mark.parametrize("qkind", ["q_absmax", "q_sabsmax", "q_mean"])
@pytest.mark.parametrize("variant", ["vfa", "vsa"])
def test_blockwise_query_repr_m_init(qkind, variant):
    # block-wise m-init seeds (src/vfa.py:104-106) on the GPU against the oracle, GQA + batch
    from paper_2604_12798_b200.api import NormalizerUnderflowError
    B, Hq, Hkv, L, d = 2, 4, 2, 1024, 128
    q, k, v = _rand((B, Hq, L, d), 151), _rand((B, Hkv, L, d), 152), _rand((B, Hkv, L, d), 153)
    kw = dict(variant=variant, causal=True, qkind=qkind)
    if variant == "vsa":
        kw["lam"] = 1e-3
    errors = [vo.forward_head(_f64(q[b, h]), _f64(k[b, h // 2]), _f64(v[b, h // 2]), q_block=128,
                              k_block=128, raise_errors=False, **kw).error
              for b in range(B) for h in range(Hq)]
    if any(e is not None for e in errors):
        # a block-wise absmax seed overestimates every row's max; VSA then skips every block
        # of some query tile and the normalizer underflows -- the reference raises, so must we
        assert variant == "vsa" and qkind != "q_mean"
        from paper_2604_12798_b200 import attention_forward
        with pytest.raises(NormalizerUnderflowError):
            attention_forward(q, k, v, **kw)
        return
    out, lse, _, st = _run_gpu(q, k, v, **kw)
    ref_o, ref_lse, ref_st = vo.forward(_f64(q), _f64(k), _f64(v), q_block=128, k_block=128, **kw)
    _compare(out, lse, ref_o, ref_lse, str(kw))
    if variant == "vfa":
        assert (st["special"], st["frozen"], st["visited"]) == (ref_st["special"], ref_st["frozen"],
                                                                ref_st["visited"])


def test_incremental_krepr_range_matches_full():
    # append-only K cache: recomputing only the tail blocks reproduces the full representations
    import ctypes
    from paper_2604_12798_b200 import _lib
    from paper_2604_12798_b200.api import _params
    lib = _lib.load()
    k = _rand((1, 2, 2048, 128), 161)
    p = _params(k.new_empty((1, 2, 2048, 128)), k, k, k, variant="vfa", causal=True, q_block=128, k_block=128,
                scale=None, kind="sabsmax", qkind="row_wise", reorder=True, use_m_init=True, tc1=None,
                n_sink=1, n_local=1, lam=None, monitor=False)
    full = torch.empty((1, 2, 16, 128), dtype=torch.bfloat16, device="cuda")
    part = torch.zeros_like(full)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert lib.vfa_krepr(ctypes.byref(p), k.data_ptr(), full.data_ptr(), st) == 0
    k2 = k.clone()
    k2[:, :, 1500:] = _rand((1, 2, 548, 128), 162)  # tokens appended after position 1500
    assert lib.vfa_krepr(ctypes.byref(p), k.data_ptr(), part.data_ptr(), st) == 0
    assert lib.vfa_krepr_range(ctypes.byref(p), k2.data_ptr(), part.data_ptr(), 1500 // 128, st) == 0
    assert lib.vfa_krepr(ctypes.byref(p), k2.data_ptr(), full.data_ptr(), st) == 0
    torch.cuda.synchronize()
    assert torch.equal(part, full)


@pytest.mark.parametrize("variant,extra", [("vfa", {}), ("blasst_fa4", dict(lam=1e-3, tau=2.0)),
                                           ("vsa", dict(lam=1e-2))])
def test_vft1_run_backend_matches_reference_report(variant, extra, tmp_path):
    # `run` on a VFT1 dump through the GPU backend: counters / stats integer-equal to the
    # report the reference CLI wrote for the same dump (tests/golden/make_vft1.py), O vs oracle
    import json
    import os

    from paper_2604_12798_b200 import runner, vft1
    fix = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "vft1")
    ref = json.load(open(os.path.join(fix, f"ref_run_{variant}.json")))
    rep = runner.run(fix, variant=variant, q_block=128, k_block=64, causal=True, out=tmp_path / "o.vft",
                     report=tmp_path / "r.json", **extra)
    assert json.load(open(tmp_path / "r.json"))["values"]["output_shape"] == [256, 64]
    assert rep["counters"] == ref["counters"]
    if ref["stats"] is not None:
        assert rep["stats"] == ref["stats"]
    q, k, v = runner.load_tensors(fix)
    kw = {"lam": extra.get("lam"), "tau": extra.get("tau", 0.0)} if variant != "vfa" else {}
    r = vo.forward_head(q, k, v, variant=variant, causal=True, q_block=128, k_block=64, **kw)
    o = vft1.read_matrix(tmp_path / "o.vft")
    assert vo.max_rel_err(o, r.out) <= O_REL
    cmp = runner.compare(fix, "fa", variant=variant, q_block=128, k_block=64, causal=True, **extra)
    assert cmp["values"]["max_rel_diff"] <= 5e-2 and set(cmp["values"]["counter_delta"]) == set(ref["counters"])


def test_module_cli_run(tmp_path):
    import os
    import subprocess
    import sys
    fix = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "vft1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "paper_2604_12798_b200", "run", "--data", fix, "--variant", "vfa",
                        "--causal", "--report", str(tmp_path / "r.json")], cwd=root, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([sys.executable, "-m", "paper_2604_12798_b200", "run", "--data", str(tmp_path),
                        "--variant", "vfa"], cwd=root, capture_output=True, text=True)
    assert r.returncode == 3  # missing q.vft -> DataError (src/cli.py:69-72)


@pytest.mark.parametrize("ranks", [2, 3])
def test_bench_sharded_path_two_ranks(ranks):
    # bench.py under torchrun with 2 / 3 ranks sharing GPU 0 (gloo): (batch, KV head) unit shards
    # (3 ranks over the tiny config's 4 units: uneven, padded gather), max-over-ranks timing,
    # NCCL-style gather + bitwise verification against the single-GPU run
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, VFA_BENCH_SHARE_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(ranks),
                        "--master-addr", "127.0.0.1", "--master-port", str(29611 + ranks), "bench.py", "--gpus", str(ranks),
                        "--config", "tiny", "--steps", "2", "--warmup", "3", "--no-cpu", "--e2e-steps", "1"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == ranks and line["verified_vs_single_gpu"] is True
    assert line["e2e"]["bitwise_equal_to_device_run"] is True


@pytest.mark.parametrize("variant", ["fa", "vfa", "vsa", "blasst", "blasst_fa4", "blasst_rowskip"])
@pytest.mark.parametrize("geom", [dict(B=2, Hq=6, Hkv=3, Lq=512, Lk=768, causal=False),
                                  dict(B=1, Hq=3, Hkv=1, Lq=768, Lk=768, causal=True),
                                  dict(B=1, Hq=4, Hkv=4, Lq=384, Lk=384, causal=True, k_block=64)])
def test_every_variant_on_mixed_geometries(variant, geom):
    # batch, odd GQA groups (one query tile per CTA), Lq != Lk, Bc = 64 for every variant
    g = dict(geom)
    B, Hq, Hkv, Lq, Lk = g.pop("B"), g.pop("Hq"), g.pop("Hkv"), g.pop("Lq"), g.pop("Lk")
    q, k, v = _rand((B, Hq, Lq, 64), 171), _rand((B, Hkv, Lk, 64), 172), _rand((B, Hkv, Lk, 64), 173)
    kw = dict(variant=variant, q_block=128, k_block=g.pop("k_block", 128), **g)
    if variant not in ("fa", "vfa"):
        kw["lam"] = 1e-2
    if variant == "blasst_fa4":
        kw["tau"] = 1.0
    out, lse, _, st = _run_gpu(q, k, v, **kw)
    okw = dict(kw)
    ref_o, ref_lse, ref_st = vo.forward(_f64(q), _f64(k), _f64(v), **okw)
    _compare(out, lse, ref_o, ref_lse, str(kw))
    assert st["visited"] == ref_st["visited"]



PAIR_VARIANTS = [("fa", {}), ("vfa", {}), ("vsa", dict(lam=1e-2)), ("blasst", dict(lam=1e-2)),
                 ("blasst_fa4", dict(lam=1e-2, tau=1.0)), ("blasst_rowskip", dict(lam=1e-2))]


@pytest.mark.parametrize("variant,extra", PAIR_VARIANTS, ids=[v for v, _ in PAIR_VARIANTS])
@pytest.mark.parametrize("bc", [64, 128])
@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("hq", [4, 8])
def test_cta_pair_against_oracle(variant, extra, bc, causal, hq):
    # cta_group::2 path: K/V tiles split between the two SMs' shared memory and consumed by
    # M = 256 MMAs issued by the leader CTA; GQA group 2: one query tile per CTA, group 4: two
    # per CTA (four heads per cluster). Planted sink so the skipping variants skip / elide / mask.
    B, Hq, Hkv, L, d = 1, hq, 2, 640, 128
    q, k, v = _rand((B, Hq, L, d), 211), _rand((B, Hkv, L, d), 212), _rand((B, Hkv, L, d), 213)
    if variant not in ("fa", "vfa"):
        amp = float(np.sqrt(8.0 * np.sqrt(d)))
        q[..., 0] = amp
        k[..., 0] = 0
        k[:, :, :bc, 0] = amp
    kw = dict(variant=variant, causal=causal, q_block=128, k_block=bc, **extra)
    okw = dict(kw)
    if variant.startswith("blasst"):
        kw["reorder"] = False
    out, lse, _, st = _run_gpu(q, k, v, cta_pair=2, **kw)
    qf, kf, vf = _f64(q), _f64(k), _f64(v)
    o_ref, l_ref = np.empty(out.shape), np.empty(lse.shape)
    visited = 0
    for h in range(Hq):
        r = vo.forward_head(qf[0, h], kf[0, h // (Hq // Hkv)], vf[0, h // (Hq // Hkv)], **okw)
        o_ref[0, h], l_ref[0, h] = r.out, r.lse
        visited += r.visited
    _compare(out, lse, o_ref, l_ref, f"{kw} pair")
    assert st["visited"] == visited
    # the pair and single-CTA paths take identical skip decisions
    out1, lse1, _, st1 = _run_gpu(q, k, v, cta_pair=1, softmax_split=4, **kw)
    assert st == st1
    if variant == "vfa":  # frozen max: same per-row arithmetic in both layouts
        assert torch.equal(out, out1) and torch.equal(lse, lse1)


def test_cta_pair_falls_back_where_ineligible():
    # odd GQA groups and d = 64 cannot pair: cta_pair = 2 runs the single-CTA kernel there
    for (hq, hkv, d) in [(3, 1, 128), (2, 1, 64)]:
        q, k, v = _rand((1, hq, 256, d), 221), _rand((1, hkv, 256, d), 222), _rand((1, hkv, 256, d), 223)
        o2, l2, _, _ = _run_gpu(q, k, v, variant="vfa", causal=True, cta_pair=2)
        o1, l1, _, _ = _run_gpu(q, k, v, variant="vfa", causal=True, cta_pair=1)
        assert torch.equal(o1, o2) and torch.equal(l1, l2)


def test_cta_pair_rejects_bad_value():
    q, k, v = _rand((1, 2, 128, 128), 231), _rand((1, 1, 128, 128), 232), _rand((1, 1, 128, 128), 233)
    with pytest.raises(ValueError):
        _run_gpu(q, k, v, variant="vfa", causal=True, cta_pair=3)


SMALLQ = [(v, qb) for v in ("fa", "vfa", "vsa", "blasst", "blasst_fa4", "blasst_rowskip") for qb in (16, 32, 64)]


@pytest.mark.parametrize("variant,qb", SMALLQ)
@pytest.mark.parametrize("causal", [True, False])
def test_small_query_blocks_against_oracle(variant, qb, causal):
    # q_block < 128 (the reference CLI default is 64): each 128-row MMA tile holds one reference
    # query block, so the schedule, special / frozen classes and skip decisions are the
    # reference's at that block size; the idle rows never reach O, LSE or the statistics
    B, Hq, Hkv, L, d, bc = 1, 4, 2, 512, 64, 64
    q, k, v = _rand((B, Hq, L, d), 241), _rand((B, Hkv, L, d), 242), _rand((B, Hkv, L, d), 243)
    extra = {}
    if variant not in ("fa", "vfa"):
        amp = float(np.sqrt(8.0 * np.sqrt(d)))
        q[..., 0] = amp
        k[..., 0] = 0
        k[:, :, :bc, 0] = amp
        extra = dict(lam=1e-2, tau=4.0) if variant == "blasst_fa4" else dict(lam=1e-2)
    kw = dict(variant=variant, causal=causal, q_block=qb, k_block=bc, **extra)
    if variant.startswith("blasst"):
        kw["reorder"] = False
    out, lse, _, st = _run_gpu(q, k, v, monitor=True, **kw)
    okw = {key: val for key, val in kw.items() if key != "reorder"}
    qf, kf, vf = _f64(q), _f64(k), _f64(v)
    o_ref, l_ref = np.empty(out.shape), np.empty(lse.shape)
    ref = {"visited": 0, "skipped": 0, "special": 0, "frozen": 0, "elided": 0, "rows_masked": 0}
    tight = True
    for h in range(Hq):
        r = vo.forward_head(qf[0, h], kf[0, h // 2], vf[0, h // 2], record_decisions=True, **okw)
        o_ref[0, h], l_ref[0, h] = r.out, r.lse
        for key in ref:
            ref[key] += getattr(r, key)
        tight &= all(mg > 1e-3 for blk in r.decisions for (_, _, mg) in blk)
    _compare(out, lse, o_ref, l_ref, str(kw))
    assert st["visited"] == ref["visited"]
    if variant in ("fa", "vfa"):
        assert (st["special"], st["frozen"]) == (ref["special"], ref["frozen"])
    if tight:
        assert st["skipped"] == ref["skipped"]
        assert st["rows_masked"] == ref["rows_masked"]
    assert st["count_over_f32"] == 0


def test_small_query_blocks_host_pipeline_and_trace():
    # q_block 64 through the chunked host path (bitwise = device path) and the device
    # StateTrace / skip trace geometry (one entry per reference query block)
    from paper_2604_12798_b200 import attention_forward
    q, k, v = _rand((1, 4, 512, 128), 251), _rand((1, 2, 512, 128), 252), _rand((1, 2, 512, 128), 253)
    kw = dict(variant="vfa", causal=True, q_block=64, k_block=128)
    o1, l1, _ = attention_forward(q, k, v, **kw)
    o2, l2, _ = attention_forward(q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory(), **kw)
    assert torch.equal(o1.cpu(), o2) and torch.equal(l1.cpu(), l2)
    _, _, info = attention_forward(q, k, v, stab_trace=True, skip_trace=True, **kw)
    assert info["stab_block"].shape == (1, 4, 512)
    qf, kf, vf = _f64(q), _f64(k), _f64(v)
    r = vo.forward_head(qf[0, 0], kf[0, 0], vf[0, 0], **kw)
    got = info["stab_block"][0, 0].cpu().numpy()
    assert (got != r.stab).mean() <= 0.01


@pytest.mark.parametrize("variant", ["fa", "vfa", "vsa"])
@pytest.mark.parametrize("hq,hkv,b,qb,bc", [(3, 1, 2, 64, 128), (2, 2, 1, 32, 128), (4, 2, 1, 16, 64)])
def test_small_query_blocks_geometries(variant, hq, hkv, b, qb, bc):
    # small reference query blocks with d = 128, odd GQA groups (one tile per CTA), batch > 1
    L, d = 384, 128
    q, k, v = _rand((b, hq, L, d), 261), _rand((b, hkv, L, d), 262), _rand((b, hkv, L, d), 263)
    kw = dict(variant=variant, causal=True, q_block=qb, k_block=bc)
    if variant == "vsa":
        kw["lam"] = 1e-2
    out, lse, _, st = _run_gpu(q, k, v, **kw)
    ref_o, ref_lse, ref_st = vo.forward(_f64(q), _f64(k), _f64(v), **kw)
    _compare(out, lse, ref_o, ref_lse, str(kw))
    assert st["visited"] == ref_st["visited"]
    if variant != "vsa":
        assert (st["special"], st["frozen"]) == (ref_st["special"], ref_st["frozen"])


@pytest.mark.parametrize("variant", ["fa", "vfa", "vsa", "blasst_rowskip"])
@pytest.mark.parametrize("lq,lk,qb,bc,causal", [(192, 192, 64, 64, True), (320, 320, 32, 64, True),
                                                (96, 256, 32, 128, False), (64, 64, 16, 64, True)])
def test_small_query_blocks_ragged_lengths(variant, lq, lk, qb, bc, causal):
    # lengths that are not multiples of the 128-row tile: the last tile's idle rows read past
    # the sequence (TMA zero fill) and are never stored
    d = 64
    q, k, v = _rand((1, 2, lq, d), 271), _rand((1, 1, lk, d), 272), _rand((1, 1, lk, d), 273)
    kw = dict(variant=variant, causal=causal, q_block=qb, k_block=bc)
    if variant in ("vsa", "blasst_rowskip"):
        kw["lam"] = 1e-2
    if variant.startswith("blasst"):
        kw["reorder"] = False
    out, lse, _, st = _run_gpu(q, k, v, **kw)
    okw = {key: val for key, val in kw.items() if key != "reorder"}
    ref_o, ref_lse, ref_st = vo.forward(_f64(q), _f64(k), _f64(v), **okw)
    _compare(out, lse, ref_o, ref_lse, str(kw))
    assert st["visited"] == ref_st["visited"]


@pytest.mark.parametrize("variant", ["fa", "vfa", "vsa"])
@pytest.mark.parametrize("hq", [4, 8])
def test_cta_pair_one_thread_per_row(variant, hq):
    # CTA pairs with the one-thread-per-row softmax layout (softmax_split = 1)
    B, Hkv, L, d = 1, 2, 512, 128
    q, k, v = _rand((B, hq, L, d), 281), _rand((B, Hkv, L, d), 282), _rand((B, Hkv, L, d), 283)
    kw = dict(variant=variant, causal=True, q_block=128, k_block=128)
    if variant == "vsa":
        kw["lam"] = 1e-2
    out, lse, _, st = _run_gpu(q, k, v, cta_pair=2, softmax_split=1, **kw)
    ref_o, ref_lse, ref_st = vo.forward(_f64(q), _f64(k), _f64(v), **kw)
    _compare(out, lse, ref_o, ref_lse, f"{kw} pair split 1")
    assert st["visited"] == ref_st["visited"]
    out1, _, _, _ = _run_gpu(q, k, v, cta_pair=1, softmax_split=1, **kw)
    if variant == "vfa":
        assert torch.equal(out, out1)


@pytest.mark.parametrize("variant", ["fa", "vfa"])
def test_large_shape_against_torch_sdpa(variant):
    # full-size GQA problem (L = 8192, 32 query / 8 KV heads, batch 2): the device output against
    # torch's fused attention on the same bf16 inputs (an independent fp32-accumulating kernel)
    import torch.nn.functional as F
    B, Hq, Hkv, L, d = 2, 32, 8, 8192, 128
    q, k, v = _rand((B, Hq, L, d), 291), _rand((B, Hkv, L, d), 292), _rand((B, Hkv, L, d), 293)
    out, lse, _, st = _run_gpu(q, k, v, variant=variant, causal=True)
    ref = F.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
    err = (out.float() - ref.float()).abs().max().item()
    assert err <= O_ABS, err
    assert st["visited"] == B * Hq * sum(range(1, L // 128 + 1))


# ----------------------------------------------------------------------------- headline sizes
# BASELINE.json configs[1] (C2) and configs[3] (C4): the full problem runs on the GPU; the float64
# oracle checks a sample of query blocks spread over the causal depth (query blocks are
# independent, so a sampled block is computed exactly as in the full pass).
C2_BLOCKS = (1, 2, 37, 128, 201, 256)


def _sampled_parity(q, k, v, heads, blocks, kw, tag):
    grp = q.shape[1] // k.shape[1]
    out, lse, info, st = _run_gpu(q, k, v, **kw)
    for h in heads:
        qq, kk, vv = _f64(q[0, h]), _f64(k[0, h // grp]), _f64(v[0, h // grp])
        r = vo.forward_head(qq, kk, vv, q_blocks=list(blocks), q_block=128, k_block=128, **kw)
        rows = np.concatenate([np.arange((i - 1) * 128, i * 128) for i in blocks])
        _compare(out[0, h, rows], lse[0, h, rows], r.out[rows], r.lse[rows], f"{tag} head {h}")
    return out, lse, st


@pytest.mark.parametrize("variant", ["vfa", "fa", "vsa"])
def test_c2_full_problem_sampled_oracle(variant):
    # 1 x 32 x 32768 x 128, 8 KV heads, causal, bf16 (Llama-3-8B prefill)
    L = 32768
    q, k, v = _rand((1, 32, L, 128), 1234), _rand((1, 8, L, 128), 1235), _rand((1, 8, L, 128), 1236)
    kw = dict(variant=variant, causal=True, lam=1e-2 if variant == "vsa" else None)
    out, lse, st = _sampled_parity(q, k, v, (0, 31), C2_BLOCKS, kw, f"C2 {variant}")
    t_r = L // 128
    assert st["visited"] == 32 * t_r * (t_r + 1) // 2
    if variant == "vfa":
        assert st["special"] == 32 * sum(min(2, i) for i in range(1, t_r + 1))
    assert torch.isfinite(out).all() and torch.isfinite(lse).all()


def test_c4_full_problem_sampled_oracle():
    # 1 x 32 x 131072 x 128 (BASELINE configs[3] on one GPU): two late blocks of one head
    L = 131072
    q, k, v = _rand((1, 32, L, 128), 7), _rand((1, 8, L, 128), 8), _rand((1, 8, L, 128), 9)
    kw = dict(variant="vfa", causal=True)
    out, lse, st = _sampled_parity(q, k, v, (13,), (1, 700, 1024), kw, "C4 vfa")
    assert torch.isfinite(out).all()
    t_r = L // 128
    assert st["special"] == 32 * sum(min(2, i) for i in range(1, t_r + 1))


def test_c2_planted_sink_vsa_skip_counts():
    # C3 at the C2 size: planted sink (src/tensor.py:153-165 trick), lambda = 1e-2; the device's
    # skip decisions equal the oracle's wherever its decision margin exceeds 1e-3
    from paper_2604_12798_b200 import attention_forward
    L, d = 32768, 128
    q, k, v = _rand((1, 32, L, d), 301), _rand((1, 8, L, d), 302), _rand((1, 8, L, d), 303)
    amp = float(np.sqrt(8.0 * np.sqrt(d)))
    q[..., 0] = amp
    k[..., 0] = 0
    k[:, :, :128, 0] = amp
    kw = dict(variant="vsa", causal=True, q_block=128, k_block=128, lam=1e-2)
    out, lse, info = attention_forward(q, k, v, check=False, skip_trace=True, **kw)
    trace = info["skip_trace"].cpu().numpy()
    blocks = (1, 2, 64, 200, 256)
    flips = 0
    for h in (0, 17):
        r = vo.forward_head(_f64(q[0, h]), _f64(k[0, h // 4]), _f64(v[0, h // 4]), record_decisions=True,
                            q_blocks=list(blocks), **kw)
        for i, dec in zip(blocks, r.decisions):
            for pos, (j, skip, margin) in enumerate(dec):
                g = trace[0, h, i - 1, pos]
                if margin > 1e-3:
                    assert (g == 2) == skip, (h, i, pos, j, margin)
                elif (g == 2) != skip:
                    flips += 1
        rows = np.concatenate([np.arange((i - 1) * 128, i * 128) for i in blocks])
        if flips == 0:
            _compare(out[0, h, rows], lse[0, h, rows], r.out[rows], r.lse[rows], f"C3 head {h}")
    assert flips <= 2
    skipped = (trace == 2).sum() / max((trace > 0).sum(), 1)
    assert skipped > 0.9  # the planted sink makes almost every block skippable at lambda 1e-2


# ----------------------------------------------------------------------------- head_dim 32 / k_block 32
@pytest.mark.parametrize("variant", ["fa", "vfa", "vsa", "blasst", "blasst_fa4", "blasst_rowskip"])
@pytest.mark.parametrize("qb,kb", [(64, 64), (128, 128), (128, 32), (32, 32)])
@pytest.mark.parametrize("causal", [True, False])
def test_head_dim_32(variant, qb, kb, causal):
    # d = 32 runs on the D = 64 kernels with TMA zero-filled columns (exact); the reference's
    # acceptance matrix covers d in {32, 64, 128} (tests/test_acceptance.py:37-61)
    B, Hq, Hkv, L, d = 1, 4, 2, 512, 32
    q, k, v = _rand((B, Hq, L, d), 501), _rand((B, Hkv, L, d), 502), _rand((B, Hkv, L, d), 503)
    kw = dict(variant=variant, causal=causal, q_block=qb, k_block=kb)
    if variant not in ("fa", "vfa"):
        kw["lam"] = 1e-3
    if variant == "blasst_fa4":
        kw["tau"] = 2.0
    out, lse, _, st = _run_gpu(q, k, v, **kw)
    ref_o, ref_lse, ref_st = vo.forward(_f64(q), _f64(k), _f64(v), **kw)
    _compare(out, lse, ref_o, ref_lse, str(kw))
    assert st["visited"] == ref_st["visited"]
    if variant in ("fa", "vfa"):
        assert (st["special"], st["frozen"]) == (ref_st["special"], ref_st["frozen"])


@pytest.mark.parametrize("variant", ["fa", "vfa", "vsa", "blasst_rowskip"])
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("split", [0, 1, 2, 4])
@pytest.mark.parametrize("hq", [2, 3])
def test_k_block_32(variant, d, split, hq):
    # 32-row key blocks: 2 threads per row (two query tiles) or one thread per row
    L = 640
    q, k, v = _rand((1, hq, L, d), 511), _rand((1, 1, L, d), 512), _rand((1, 1, L, d), 513)
    kw = dict(variant=variant, causal=True, q_block=128, k_block=32, softmax_split=split)
    if variant in ("vsa", "blasst_rowskip"):
        kw["lam"] = 1e-3
    out, lse, _, st = _run_gpu(q, k, v, **kw)
    kw.pop("softmax_split")
    ref_o, ref_lse, ref_st = vo.forward(_f64(q), _f64(k), _f64(v), **kw)
    _compare(out, lse, ref_o, ref_lse, str(kw))
    if variant in ("fa", "vfa"):
        assert (st["special"], st["frozen"]) == (ref_st["special"], ref_st["frozen"])


@pytest.mark.parametrize("n", [64, 256, 1024])
@pytest.mark.parametrize("d", [32, 64, 128])
@pytest.mark.parametrize("causal", [False, True])
def test_reference_acceptance_matrix(n, d, causal):
    # the reference's acceptance gate #1 problem matrix (tests/test_acceptance.py:37-61: blocks of
    # 64, n in {64, 256, 1024}, d in {32, 64, 128}) through the drop-in entry points, against the
    # exact oracle (float64 naive attention there; bf16 tolerance here)
    from paper_2604_12798_b200 import AttentionProblem, BlockSpec, fa_forward, vfa_forward
    q, k, v = _rand((n, d), 601 + n + d), _rand((n, d), 602 + n + d), _rand((n, d), 603 + n + d)
    p = AttentionProblem(q, k, v, blocks=BlockSpec(n, n, d, 64, 64), causal=causal)
    ref = vo.forward_head(_f64(q), _f64(k), _f64(v), variant="fa", causal=causal, q_block=64, k_block=64)
    for fwd in (fa_forward, vfa_forward):
        res = fwd(p)
        _compare(res[0], res.lse, ref.out, ref.lse, f"{fwd.__name__} n={n} d={d} causal={causal}")


@pytest.mark.parametrize("variant", ["vfa", "fa"])
def test_state_trace_snapshots_and_final_m(variant):
    # the reference's StateTrace records (src/core.py:35-54) from the device: per visit the running
    # max after the visit; stabilization_positions(trace, final_m) (src/analysis.py:39-78) on them
    from paper_2604_12798_b200 import AttentionProblem, BlockSpec, fa_forward, stabilization_positions, vfa_forward
    L, d = 1024, 64
    q, k, v = _rand((L, d), 701), _rand((L, d), 702), _rand((L, d), 703)
    p = AttentionProblem(q, k, v, blocks=BlockSpec(L, L, d, 128, 64), causal=True)
    res = (vfa_forward(p, n_local=2) if variant == "vfa" else fa_forward(p))
    trace = res[2]
    assert trace.snapshots is not None and trace.snapshots.shape == (L, L // 64)
    snap = trace.snapshots.double().cpu().numpy()
    ref = vo.forward_head(_f64(q), _f64(k), _f64(v), variant=variant, causal=True, q_block=128, k_block=64,
                          n_local=2 if variant == "vfa" else 1)
    # records: block order = the reference schedule; the last snapshot is the final running max
    tc = L // 64
    for bi, recs in enumerate(trace.records):
        i = bi + 1
        vmax, local = vo.visible_key_blocks(i, 128, 64, tc, True), vo.local_key_block(i, 128, 64, tc)
        order = vo.build_schedule(i, vmax, local, True, 1, 2)[0] if variant == "vfa" else tuple(range(1, vmax + 1))
        assert tuple(j for _, j, _ in recs) == tuple(order)
    final = np.array([snap[r, np.where(np.isfinite(snap[r]))[0][-1]] for r in range(L)])
    if variant == "fa":  # the running max ends at the exact row max (src/reference.py:105-111)
        exact = vo.exact_rowmax_global(_f64(q), _f64(k), 1.0 / np.sqrt(d), True)
        assert np.abs(final - exact).max() <= 1e-3
    rep0 = stabilization_positions(trace)
    rep1 = stabilization_positions(trace, final_m=final)
    assert np.array_equal(rep0.positions, rep1.positions)
    assert (rep0.positions != ref.stab).mean() <= 0.01
    with pytest.raises(ValueError):
        stabilization_positions(trace, final_m=final + 1.0)
