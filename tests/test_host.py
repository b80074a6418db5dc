"""CPU tests of the host side: the C-ABI library loads and exports every symbol the
header declares, host-side validation (no GPU), the device tile scheduler's host
mirror against the oracle, and the drop-in API's validation / op accounting."""

import ctypes
import itertools
import os
import re

import numpy as np
import pytest

from golden_io import case_names, case
from oracle import vfa_oracle as vo

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2604_12798_b200 import _lib, build
    build.build()
    return _lib.load()


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "vfa_b200.h")).read()
    return sorted(set(re.findall(r"^VFA_API\s+(?:int|size_t|const char\*)\s+(vfa_\w+)\(", txt, re.M)))


def test_library_exports_every_header_symbol(lib):
    from paper_2604_12798_b200 import _lib
    syms = _header_symbols()
    assert syms and set(syms) == set(_lib.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s
    assert b"sm_100a" in lib.vfa_version()


def test_params_struct_layout_matches_header():
    from paper_2604_12798_b200._lib import VfaParams
    # 6 int64 + 12 int64 strides + double + 12 int32 + double + 2 int32
    # + softmax_split (int32), tau (double), cta_pair + reserved (int32)
    assert ctypes.sizeof(VfaParams) == 6 * 8 + 12 * 8 + 8 + 12 * 4 + 8 + 2 * 4 + 8 + 2 * 4


def _params(**kw):
    from paper_2604_12798_b200._lib import VfaParams
    p = VfaParams()
    p.batch, p.heads_q, p.heads_kv, p.seq_q, p.seq_k, p.head_dim = 1, 4, 2, 1024, 1024, 128
    for arr in (p.q_stride, p.k_stride, p.v_stride, p.o_stride):
        arr[:] = (4 * 1024 * 128, 1024 * 128, 128)
    p.causal, p.q_block, p.k_block, p.variant = 1, 128, 128, 1
    p.kind, p.qkind, p.reorder, p.use_m_init, p.tc1 = 0, 0, 1, 1, 0
    p.n_sink, p.n_local, p.monitor, p.lam = 1, 1, 0, 0.0
    for k, v in kw.items():
        setattr(p, k, v)
    return p


@pytest.mark.parametrize("field,value,code", [
    ("variant", 7, 2), ("kind", 9, 2), ("qkind", 4, 2), ("q_block", 48, 2), ("k_block", 96, 2),
    ("head_dim", 96, 2), ("seq_q", 1000, 3), ("seq_k", 1000, 3), ("heads_q", 3, 3), ("tc1", 99, 2),
    ("n_sink", -1, 2), ("tau", -1.0, 2), ("softmax_split", 3, 2), ("variant", 6, 2),
    ("scale", -0.125, 2), ("scale", float("nan"), 2), ("scale", float("inf"), 2),
])
def test_check_params_codes(lib, field, value, code):
    assert lib.vfa_check_params(ctypes.byref(_params())) == 0
    p = _params(**{field: value})
    if field == "seq_k":
        p.causal = 0
    assert lib.vfa_check_params(ctypes.byref(p)) == code
    assert lib.vfa_last_error()


def test_check_params_causal_and_strides(lib):
    p = _params(seq_k=512)
    assert lib.vfa_check_params(ctypes.byref(p)) == 3  # causal needs Nq == Nk
    p = _params()
    p.q_stride[2] = 130
    assert lib.vfa_check_params(ctypes.byref(p)) == 3
    p = _params(variant=2, lam=1.5)
    assert lib.vfa_check_params(ctypes.byref(p)) == 2
    assert lib.vfa_workspace_bytes(ctypes.byref(_params())) >= 2 * 8 * 128 * 2


def test_status_code_mapping(lib):
    st = (ctypes.c_uint * 4)(0, 0xFFFFFFFF, 0xFFFFFFFF, 0)
    assert lib.vfa_status_code(st) == 0
    st[0], st[1] = 2, 17
    assert lib.vfa_status_code(st) == 4
    assert b"normalizer underflow at query row 17" in lib.vfa_last_error()
    st[0], st[2] = 1, 3
    assert lib.vfa_status_code(st) == 4
    assert b"fully masked" in lib.vfa_last_error()


GEOMS = [(128, 128), (128, 64), (64, 64), (128, 32), (32, 128)]


@pytest.mark.parametrize("qb,kb", GEOMS)
@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("ns,nl", [(1, 1), (1, 2), (2, 2), (0, 1), (3, 0), (2, 3)])
@pytest.mark.parametrize("reorder", [True, False])
def test_device_scheduler_matches_oracle(lib, qb, kb, causal, ns, nl, reorder):
    from paper_2604_12798_b200 import tile_schedule
    L = 1024
    t_r, t_c = L // qb, L // kb
    for i in range(1, t_r + 1):
        vmax = vo.visible_key_blocks(i, qb, kb, t_c, causal)
        local = vo.local_key_block(i, qb, kb, t_c)
        ref = vo.build_schedule(i, vmax, local, reorder, ns, nl)
        assert tile_schedule(i, qb, kb, t_c, causal, ns, nl, reorder) == ref, i
        order, special = tile_schedule(i, qb, kb, t_c, causal, ns, nl, reorder, variant="fa")
        assert order == tuple(range(1, vmax + 1)) and special == frozenset(order)


def test_reference_schedule_known_answers(lib):
    # tests/test_vfa.py:60-77, expressed through geometry (Br = Bc = 1 block units)
    from paper_2604_12798_b200 import tile_schedule
    assert tile_schedule(3, 1, 1, 5, False) == ((1, 3, 2, 4, 5), frozenset({1, 3}))
    assert tile_schedule(1, 1, 1, 4, False) == ((1, 2, 3, 4), frozenset({1}))
    assert tile_schedule(3, 1, 1, 5, False, reorder=False) == ((1, 2, 3, 4, 5), frozenset({1, 3}))
    # local beyond the visible range (vmax = 2, local = 5 is impossible with causal; use Tc)
    assert tile_schedule(5, 1, 1, 2, False) == ((1, 2), frozenset({1, 2}))


@pytest.mark.parametrize("name", case_names())
def test_op_counters_integer_equal_reference(name):
    """OpCounters charged from per-class block counts equal the reference counters."""
    from paper_2604_12798_b200.api import OpCounters
    m, q, k, v, _, _ = case(name)
    if "counters.blocks_processed" not in m or m["error"]:
        pytest.skip("no counters recorded")
    kw = {key: m[key] for key in ("kind", "qkind", "reorder", "use_m_init", "tc1", "lam", "tau", "order") if key in m}
    r = vo.forward_head(q, k, v, variant=m["variant"], causal=m["causal"], q_block=m["q_block"],
                        k_block=m["k_block"], n_sink=m["n_sink"], n_local=m["n_local"], **kw)
    st = dict(visited=r.visited, skipped=r.skipped, special=r.special, frozen=r.frozen,
              elided=r.elided, rows_masked=r.rows_masked)
    c = OpCounters.from_stats(m["variant"], st, m["q_block"], m["k_block"], q.shape[1])
    for f, val in c.as_dict().items():
        assert val == m[f"counters.{f}"], f


def test_api_validation_without_gpu():
    from paper_2604_12798_b200 import AttentionProblem, BlockSpec, SkipConfig
    with pytest.raises(ValueError):
        BlockSpec(100, 100, 64, 64, 64)
    with pytest.raises(ValueError):
        SkipConfig(lam=0.0)
    with pytest.raises(ValueError):
        SkipConfig(lam=0.5, granularity="tile")
    assert SkipConfig(lam=None).ln_lambda == float("-inf")
    z = np.zeros((256, 64))
    with pytest.raises(ValueError):
        AttentionProblem(z, np.zeros((128, 64)), np.zeros((128, 64)), causal=True)
    with pytest.raises(ValueError):
        AttentionProblem(z, np.zeros((256, 32)), np.zeros((256, 32)))
    with pytest.raises(ValueError):
        AttentionProblem(z, z, z, blocks=BlockSpec(512, 512, 64, 128, 128))


def test_tensor_validation_without_gpu():
    # shape mismatches must raise ValueError before any pointer crosses the C ABI (the C side
    # takes batch / head_dim from q and the key length from k)
    import torch
    from paper_2604_12798_b200 import attention_forward_host
    from paper_2604_12798_b200.api import _check_outputs, _params
    bf = torch.bfloat16
    q = torch.zeros(1, 4, 256, 64, dtype=bf)
    k = torch.zeros(1, 2, 256, 64, dtype=bf)
    for kk, vv, msg in ((k, torch.zeros(1, 2, 128, 64, dtype=bf), "same shape"),
                        (torch.zeros(2, 2, 256, 64, dtype=bf),) * 2 + ("batch",),
                        (torch.zeros(1, 2, 256, 32, dtype=bf),) * 2 + ("head dimension",),
                        (torch.zeros(1, 3, 256, 64, dtype=bf),) * 2 + ("multiple",)):
        with pytest.raises(ValueError, match=msg):
            attention_forward_host(q, kk, vv, variant="vfa", causal=True)
    with pytest.raises(ValueError, match="out must have"):
        _check_outputs(q, torch.zeros(1, 4, 128, 64, dtype=bf), torch.zeros(1, 4, 256), q.device)
    with pytest.raises(ValueError, match="lse"):
        _check_outputs(q, torch.zeros_like(q), torch.zeros(1, 4, 256, dtype=torch.float64), q.device)
    _check_outputs(q, torch.zeros_like(q), torch.zeros(1, 4, 256), q.device)
    kw = dict(variant="vfa", causal=True, q_block=128, k_block=128, kind="sabsmax", qkind="row_wise",
              reorder=True, use_m_init=True, tc1=None, n_sink=1, n_local=1, lam=None, monitor=False)
    for bad in (0.0, -0.5, float("nan")):  # an explicit scale is never silently replaced
        with pytest.raises(ValueError, match="scale"):
            _params(q, k, k, q, scale=bad, **kw)
    assert _params(q, k, k, q, scale=None, **kw).scale == 0.0
    assert _params(q, k, k, q, scale=0.3, **kw).scale == 0.3


def test_stat_float_keys_roundtrip():
    import struct
    from paper_2604_12798_b200 import _lib

    def key(f):  # the kernel's float_key
        u = struct.unpack("<I", struct.pack("<f", f))[0]
        return (~u & 0xFFFFFFFF) if u & 0x80000000 else (u | 0x80000000)

    vals = [-1e30, -100.0, -1.5, -0.0, 0.0, 1e-30, 2.5, 127.9, 3e38]
    keys = [key(v) for v in vals]
    assert keys == sorted(keys)  # order preserving
    for v in vals:
        assert _lib.key_to_float(key(v)) == np.float32(v)
    assert np.isnan(_lib.key_to_float(0))


def test_entry_points_fail_loudly_without_library(monkeypatch, tmp_path):
    from paper_2604_12798_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(_lib.LibraryNotBuilt):
        _lib.load()


def test_host_scratch_bytes(lib):
    p = _params()  # B=1, Hq=4, Hkv=2 (GQA group 2), L=1024, d=128
    one = lib.vfa_host_scratch_bytes(ctypes.byref(p), 1, 0)
    two = lib.vfa_host_scratch_bytes(ctypes.byref(p), 2, 0)
    sub = lib.vfa_host_scratch_bytes(ctypes.byref(p), 1, 1)
    # K/V slots (2 x [K, V, representations] of one KV head) + Q/O/LSE slots (2 query heads)
    kv_slot = 2 * (1024 * 128 * 2)
    q_slot = 2 * (2 * 1024 * 128 * 2) + 2 * 1024 * 4
    assert one >= 2 * kv_slot + 2 * q_slot  # 2 groups -> 2 K/V slots, 2 chunks -> 2 Q slots
    assert two >= kv_slot * 2 and sub < one * 2
    assert lib.vfa_host_scratch_bytes(ctypes.byref(p), 3, 0) == 0  # 3 does not divide Hkv = 2
    assert lib.vfa_host_scratch_bytes(ctypes.byref(p), 0, 0) == 0
    assert lib.vfa_host_scratch_bytes(ctypes.byref(p), 2, 1) == 0  # query sub-chunks need 1 KV head
    assert lib.vfa_host_scratch_bytes(ctypes.byref(_params(k_block=96)), 1, 0) == 0


@pytest.mark.parametrize("name", [n for n in case_names() if "stab.frac_sink" in case(n)[0]])
def test_stabilization_report_matches_reference(name):
    # api.stabilization_positions on the reference's own positions reproduces its fractions
    import torch
    from golden_io import case_stab
    from paper_2604_12798_b200.api import BlockSpec, DeviceTrace, stabilization_positions
    m, q, *_ = case(name)
    b = BlockSpec(q.shape[0], q.shape[0], q.shape[1], m["q_block"], m["k_block"])
    local = [min((i * b.q_block - 1) // b.k_block + 1, b.t_c) for i in range(1, b.t_r + 1)]
    rep = stabilization_positions(DeviceTrace(b.q_block, torch.from_numpy(case_stab(name)), local))
    assert rep.frac_sink == m["stab.frac_sink"] and rep.frac_local == m["stab.frac_local"]
    assert rep.frac_other == m["stab.frac_other"]


@pytest.mark.parametrize("variant", ["fa", "vfa", "blasst", "blasst_fa4", "blasst_rowskip"])
@pytest.mark.parametrize("reorder", [True, False])
def test_host_schedule_mirror_matches_oracle(variant, reorder):
    # vfa_schedule (the device scheduler's host mirror) == the oracle's visit order / exact set
    from paper_2604_12798_b200 import build, tile_schedule
    build.build()
    qb, kb, tc = 128, 64, 16
    for i in range(1, 9):
        order, special = tile_schedule(i, qb, kb, tc, True, reorder=reorder, variant=variant)
        vmax = vo.visible_key_blocks(i, qb, kb, tc, True)
        local = vo.local_key_block(i, qb, kb, tc)
        if variant == "fa" or variant in ("blasst_fa4", "blasst_rowskip") or (variant == "blasst" and not reorder):
            ref_order, ref_special = tuple(range(1, vmax + 1)), frozenset(range(1, vmax + 1))
        elif variant == "blasst":
            ref_order, _ = vo.build_schedule(i, vmax, local, True)
            ref_special = frozenset(range(1, vmax + 1))
        else:
            ref_order, ref_special = vo.build_schedule(i, vmax, local, reorder)
        assert order == tuple(ref_order) and special == frozenset(ref_special), (variant, i)
