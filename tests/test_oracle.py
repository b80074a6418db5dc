"""Pin the CPU oracle (oracle/vfa_oracle.py) before it is trusted as the checker.

1. Bit-for-bit against the reference package's own outputs on every golden case
   (tests/golden/make_golden.py ran vfa_lab itself).
2. The reference's known-answer tests for this path (tests/test_vfa.py,
   tests/test_sparse.py, tests/test_acceptance.py of /root/reference/pkg).
"""

import hashlib

import numpy as np
import pytest

from golden_io import case, case_names, case_stab
from oracle import vfa_oracle as vo


def _kw(m):
    kw = dict(variant=m["variant"], causal=m["causal"], q_block=m["q_block"],
              k_block=m["k_block"], n_sink=m["n_sink"], n_local=m["n_local"],
              raise_errors=False)
    for key in ("kind", "qkind", "reorder", "use_m_init", "tc1", "lam", "tau", "order"):
        if key in m:
            kw[key] = m[key]
    return kw


@pytest.mark.parametrize("name", case_names())
def test_oracle_bitwise_equals_reference(name):
    m, q, k, v, out32, lse = case(name)
    r = vo.forward_head(q, k, v, monitor=True, **_kw(m))
    if m["error"]:
        kind, row = m["error"].split(":")
        assert r.error is not None
        assert type(r.error).__name__.replace("Row", "RowError").replace(
            "Underflow", "UnderflowError") == kind
        assert r.error.row == int(row)
        return
    assert r.error is None
    digest = hashlib.sha256(np.ascontiguousarray(r.out, dtype=np.float64).tobytes()).hexdigest()
    assert digest == m["out_sha256"], "oracle O differs bitwise from the reference"
    assert np.array_equal(r.lse, lse)
    if "stats.blocks_visited" in m:
        assert r.visited == m["stats.blocks_visited"]
        assert r.skipped == m["stats.blocks_skipped"]
        if m["variant"] == "vsa":
            assert r.special == m["stats.processed_special"]
            assert r.frozen == m["stats.processed_frozen"]
        if "stats.blocks_processed" in m:
            assert r.special + r.frozen == m["stats.blocks_processed"]
            assert r.elided == m["stats.rescales_elided"]
            assert r.rows_masked == m["stats.rows_masked"]
    if "counters.rowmax_reductions" in m and m["variant"] in ("fa", "vfa"):
        assert r.special == m["counters.rescale_events"]
    if "mon.count_over_f32" in m:
        assert r.monitor.count_over_f32 == m["mon.count_over_f32"]
        assert r.monitor.count_over_f16 == m["mon.count_over_f16"]
        assert r.monitor.exp_arg_max == m["mon.exp_arg_max"]
    if "mon.gap.min" in m:  # OverflowMonitor.record_gap (src/vfa.py:129-135), bit-for-bit
        for key in ("min", "max", "mean", "frac_below"):
            assert r.monitor.calibration_gap[key] == m[f"mon.gap.{key}"], key
    else:
        assert r.monitor.calibration_gap is None or m["variant"] not in ("vfa", "vsa")
    stab = case_stab(name)
    if stab is not None:  # StateTrace -> stabilization_positions (src/analysis.py:39-78)
        assert np.array_equal(r.stab, stab)


def test_sabsmax_known_answers():
    # reference tests/test_vfa.py:35-41
    assert np.array_equal(vo.sabsmax(np.array([[3.0, -2.0], [-3.0, 2.0]])), [3.0, -2.0])
    assert np.array_equal(vo.sabsmax(np.array([[1.0, -5.0], [-4.0, 2.0]])), [-4.0, -5.0])
    row = np.array([[0.3, -1.7, 0.0]])
    assert np.array_equal(vo.sabsmax(row), row[0])


def test_block_repr_known_answers():
    # reference tests/test_vfa.py:128-137
    b = np.array([[1.0, -3.0], [2.0, 1.0]])
    assert np.array_equal(vo.block_repr(b, "sabsmax"), [2.0, -3.0])
    assert np.array_equal(vo.block_repr(b, "k_max"), [2.0, 1.0])
    assert np.array_equal(vo.block_repr(b, "k_mean"), [1.5, -1.0])
    assert np.array_equal(vo.block_repr(b, "k_absmax_unsigned"), [2.0, 3.0])
    with pytest.raises(ValueError):
        vo.block_repr(b, "median")


def test_schedule_known_answers():
    # reference tests/test_vfa.py:60-77
    assert vo.build_schedule(3, 5, 3, True) == ((1, 3, 2, 4, 5), frozenset({1, 3}))
    assert vo.build_schedule(1, 4, 1, True) == ((1, 2, 3, 4), frozenset({1}))
    assert vo.build_schedule(5, 2, 5, True) == ((1, 2), frozenset({1}))
    assert vo.build_schedule(3, 5, 3, False) == ((1, 2, 3, 4, 5), frozenset({1, 3}))
    # generalisation: 1 sink + 2 local
    assert vo.build_schedule(4, 6, 4, True, 1, 2) == ((1, 3, 4, 2, 5, 6), frozenset({1, 3, 4}))
    assert vo.build_schedule(2, 2, 2, True, 1, 2) == ((1, 2), frozenset({1, 2}))


def test_m_init_exact_on_constant_key_block():
    # reference tests/test_vfa.py:145-154
    rng = np.random.default_rng(30)
    qi = rng.normal(size=(8, 4))
    key_row = rng.normal(size=4)
    assert np.array_equal(vo.m_init(qi, [key_row.copy()], 0.5), 0.5 * (qi @ key_row))


def test_rowmax_events_law():
    # reference tests/test_vfa.py:79-85 and tests/test_acceptance.py:82-95:
    # causal VFA at Br == Bc does min(2, i) exact updates per query block.
    rng = np.random.default_rng(0)
    n, d, b = 512, 16, 64
    q, k, v = (rng.normal(size=(n, d)) for _ in range(3))
    r = vo.forward_head(q, k, v, variant="vfa", causal=True, q_block=b, k_block=b)
    t_r = n // b
    assert r.special == sum(min(2, i) for i in range(1, t_r + 1))
    assert r.special + r.frozen == sum(range(1, t_r + 1))
    # C1: 1 sink + 2 local at L=1024/B=64 gives 45 exact updates (31 at (1,1))
    n = 1024
    q, k, v = (rng.normal(size=(n, d)) for _ in range(3))
    r2 = vo.forward_head(q, k, v, variant="vfa", causal=True, q_block=64, k_block=64, n_local=2)
    assert r2.special == 45
    r1 = vo.forward_head(q, k, v, variant="vfa", causal=True, q_block=64, k_block=64)
    assert r1.special == 31


def test_vfa_matches_naive_and_fa():
    rng = np.random.default_rng(1)
    n, d = 256, 32
    q, k, v = (rng.normal(size=(n, d)) for _ in range(3))
    s = (q @ k.T) / np.sqrt(d)
    s[np.triu_indices(n, 1)] = -np.inf
    w = np.exp(s - s.max(1, keepdims=True))
    naive = (w / w.sum(1, keepdims=True)) @ v
    for variant in ("fa", "vfa", "vsa"):
        r = vo.forward_head(q, k, v, variant=variant, causal=True, q_block=64, k_block=64,
                            lam=1e-9 if variant == "vsa" else None)
        assert vo.max_rel_err(r.out, naive) <= 1e-10
        lse = np.log(np.exp(s - s.max(1, keepdims=True)).sum(1)) + s.max(1)
        assert np.abs(r.lse - lse).max() <= 1e-12


def test_vsa_tiny_lambda_bitwise_vfa():
    # reference tests/test_sparse.py:148-153
    rng = np.random.default_rng(3)
    q, k, v = (rng.normal(size=(256, 32)) for _ in range(3))
    a = vo.forward_head(q, k, v, variant="vfa", q_block=64, k_block=64)
    b = vo.forward_head(q, k, v, variant="vsa", q_block=64, k_block=64, lam=1e-9)
    assert b.skipped == 0
    assert np.array_equal(a.out, b.out)


def test_gqa_batching_maps_heads():
    rng = np.random.default_rng(4)
    q = rng.normal(size=(1, 4, 128, 16))
    k = rng.normal(size=(1, 2, 128, 16))
    v = rng.normal(size=(1, 2, 128, 16))
    out, lse, st = vo.forward(q, k, v, variant="vfa", causal=True, q_block=32, k_block=32)
    for h in range(4):
        r = vo.forward_head(q[0, h], k[0, h // 2], v[0, h // 2], variant="vfa", causal=True,
                            q_block=32, k_block=32)
        assert np.array_equal(out[0, h], r.out)
    assert st["visited"] == 4 * sum(range(1, 5))


def test_errors_and_validation():
    with pytest.raises(ValueError):
        vo.forward_head(np.zeros((100, 8)), np.zeros((100, 8)), np.zeros((100, 8)), q_block=64)
    with pytest.raises(ValueError):
        vo.forward_head(np.zeros((64, 8)), np.zeros((64, 8)), np.zeros((64, 8)),
                        variant="vsa", q_block=64, k_block=64, lam=1.5)
    with pytest.raises(ValueError):
        vo.forward_head(np.zeros((64, 8)), np.zeros((64, 8)), np.zeros((64, 8)), variant="x")
