"""CPU oracle for the VFA / VSA / FA attention forward pass — TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference `vfa_lab` algorithms
(arXiv 2604.12798, /root/reference/pkg/src/vfa_lab). It exists to CHECK the B200
kernels: only `tests/`, `__graft_entry__.smoke()` and the `cpu_baseline` /
`--impl reference` legs of `bench.py` may import it. The product path
(`paper_2604_12798_b200`) never calls it and has no CPU fallback.

Parity pinning: `tests/golden/*.npz` were produced by running the reference package
itself on the same (bf16-rounded) inputs (`tests/golden/make_golden.py`); the CPU
test-suite asserts this restatement reproduces those outputs BIT-FOR-BIT (the same
float64 expressions in the same order, same BLAS shapes), plus the reference's own
known-answer tests (sabsmax / block_repr / schedule / counter laws).

Extensions over the reference (each reduces to the reference at its default):
  * LSE output  lse = m + log(l) captured at finalize (reference never returns it).
  * (n_sink, n_local) schedule generalisation; (1, 1) is the reference schedule.
  * [B, H, L, d] batching with grouped-query attention (kv head = h // (Hq/Hkv)).
  * per-(q-block, visit) skip decisions and their decision margin, for VSA parity.

Citations are `src/X.py:N` = /root/reference/pkg/src/vfa_lab/X.py line N.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

NEG_INF = float("-inf")
KEY_REPRS = ("sabsmax", "k_max", "k_mean", "k_absmax_unsigned")  # src/vfa.py:39
QUERY_REPRS = ("row_wise", "q_absmax", "q_sabsmax", "q_mean")  # src/vfa.py:40
F16_EXP_LIMIT = float(np.log(65504.0))  # src/vfa.py:43
F32_EXP_LIMIT = 88.7228  # src/vfa.py:44


class FullyMaskedRow(Exception):
    """Mirror of FullyMaskedRowError (src/errors.py:4-9)."""

    def __init__(self, row):
        self.row = row
        super().__init__(f"query row {row} is fully masked; cannot normalize")


class NormalizerUnderflow(Exception):
    """Mirror of NormalizerUnderflowError (src/errors.py:12-17)."""

    def __init__(self, row):
        self.row = row
        super().__init__(f"normalizer underflow at query row {row}")


# ----------------------------------------------------------------------------- geometry
def visible_key_blocks(i: int, qb: int, kb: int, t_c: int, causal: bool) -> int:
    """src/core.py:112-117 — highest visible key block (1-based) for query block i."""
    if not causal:
        return t_c
    return min((i * qb - 1) // kb + 1, t_c)


def local_key_block(i: int, qb: int, kb: int, t_c: int) -> int:
    """src/core.py:120-122 — key block aligned with query block i."""
    return min((i * qb - 1) // kb + 1, t_c)


def special_blocks(vmax: int, local: int, n_sink: int = 1, n_local: int = 1) -> list:
    """Exact-update (rowmax + rescale) block set, ascending.

    src/vfa.py:146 gives {1, local} & [1..vmax]; generalised to the first n_sink blocks
    plus the n_local blocks ending at `local`.
    """
    s = set(range(1, n_sink + 1)) | set(range(local - n_local + 1, local + 1))
    return sorted(j for j in s if 1 <= j <= vmax)


def build_schedule(i: int, vmax: int, local: int, reorder: bool,
                   n_sink: int = 1, n_local: int = 1):
    """src/vfa.py:146-153 generalised: returns (order tuple, special frozenset).

    reorder: specials first (ascending), then the remaining blocks ascending.
    At (n_sink, n_local) = (1, 1) this is exactly the reference: head [1] or [1, local],
    tail [2..vmax] minus local (src/vfa.py:151-153; SPEC.md:301 for i = 1).
    """
    spec = special_blocks(vmax, local, n_sink, n_local)
    if not reorder:
        return tuple(range(1, vmax + 1)), frozenset(spec)
    sset = set(spec)
    tail = [j for j in range(1, vmax + 1) if j not in sset]
    return tuple(spec + tail), frozenset(spec)


# ----------------------------------------------------------------------------- representations
def sabsmax(block: np.ndarray) -> np.ndarray:
    """src/vfa.py:47-53: per column, the entry of largest |.|, sign kept, first row on ties."""
    idx = np.argmax(np.abs(block), axis=0)
    return block[idx, np.arange(block.shape[1])]


def block_repr(block: np.ndarray, kind: str) -> np.ndarray:
    """src/vfa.py:56-66."""
    if kind == "sabsmax":
        return sabsmax(block)
    if kind == "k_max":
        return block.max(axis=0)
    if kind == "k_mean":
        return block.mean(axis=0)
    if kind == "k_absmax_unsigned":
        return np.abs(block).max(axis=0)
    raise ValueError(f"unknown key representation {kind!r}")


def query_repr(block: np.ndarray, kind: str) -> np.ndarray:
    """src/vfa.py:69-76."""
    if kind == "q_sabsmax":
        return sabsmax(block)
    if kind == "q_absmax":
        return np.abs(block).max(axis=0)
    if kind == "q_mean":
        return block.mean(axis=0)
    raise ValueError(f"unknown query representation {kind!r}")


def precompute_kreprs(k: np.ndarray, kb: int, kind: str, tc1: int | None = None) -> list:
    """src/vfa.py:79-88: one representation per key block j <= tc1 (default all)."""
    t_c = k.shape[0] // kb
    tc1 = t_c if tc1 is None else tc1
    if not (1 <= tc1 <= t_c):
        raise ValueError(f"tc1 must be in 1..{t_c}, got {tc1}")
    return [block_repr(k[(j - 1) * kb: j * kb], kind) for j in range(1, tc1 + 1)]


def m_init(qi: np.ndarray, kreprs: list, scale: float, qkind: str = "row_wise") -> np.ndarray:
    """src/vfa.py:91-106: seed of the running max for one query block."""
    if not kreprs:
        raise ValueError("kreprs must be nonempty")
    if qkind == "row_wise":
        return np.stack([scale * (qi @ kr) for kr in kreprs]).max(axis=0)
    qr = query_repr(qi, qkind)
    best = max(scale * float(qr @ kr) for kr in kreprs)
    return np.full(qi.shape[0], best)


# ----------------------------------------------------------------------------- tile primitives
def tile_scores(q, k, scale, causal, i, j, qb, kb):
    """src/reference.py:83-97: scaled, entrywise-causally-masked score tile (1-based i, j)."""
    qi = q[(i - 1) * qb: i * qb]
    kj = k[(j - 1) * kb: j * kb]
    s = (qi @ kj.T) * scale
    if causal:
        rows = (i - 1) * qb + np.arange(qb)
        cols = (j - 1) * kb + np.arange(kb)
        s[cols[None, :] > rows[:, None]] = NEG_INF
    return s


def _rowsum(x):
    """src/tensor.py:81-89: strictly left-to-right per-row accumulation."""
    return np.cumsum(x, axis=1)[:, -1]


def _exp_args(s, m):
    """src/core.py:67-73: S - m with masked entries kept at -inf."""
    arg = s - m[:, None]
    masked = np.isneginf(s)
    if masked.any():
        arg[masked] = NEG_INF
    return arg


def _rescale_factor(m_old, m_new):
    """src/core.py:76-83: exp(m_old - m_new), 1 where m_new is still -inf."""
    dead = np.isneginf(m_new)
    with np.errstate(invalid="ignore"):
        f = np.exp(m_old - m_new)
    if dead.any():
        f[dead] = 1.0
    return f


def _tile_skippable(m_tilde, m_merged, ln_lambda):
    """src/sparse.py:99-109: every row strictly below threshold; dead rows pass unless -inf."""
    with np.errstate(invalid="ignore"):
        below = (m_tilde - m_merged) < ln_lambda
    dead = np.isneginf(m_tilde) & np.isneginf(m_merged)
    if ln_lambda != NEG_INF:
        below |= dead
    return bool(np.all(below))


def _skip_margin(m_tilde, m_merged, ln_lambda):
    """Distance of the all-rows skip decision from its threshold (inf when undecidable)."""
    if ln_lambda == NEG_INF:
        return math.inf
    with np.errstate(invalid="ignore"):
        g = m_tilde - m_merged
    g = g[np.isfinite(g)]
    if g.size == 0:
        return math.inf
    return abs(float(g.max()) - ln_lambda)


# arguments within this distance (natural units) of a monitor threshold are "near": an fp32
# device computes the argument with error well below it, so its counts may differ from the
# float64 ones by at most the near counts (test infrastructure, not in the reference)
NEAR_MARGIN = 5e-3


@dataclass
class Monitor:
    """src/vfa.py:109-135 (OverflowMonitor.record / record_gap)."""

    exp_arg_max: float = NEG_INF
    count_over_f16: int = 0
    count_over_f32: int = 0
    near_f16: int = 0
    near_f32: int = 0
    calibration_gap: dict | None = None
    gap: np.ndarray | None = None  # per-row m seed - exact global row max (record_gap input)

    def record(self, args):
        finite = args[~np.isneginf(args)]
        if finite.size == 0:
            return
        self.exp_arg_max = max(self.exp_arg_max, float(finite.max()))
        self.count_over_f16 += int((finite > F16_EXP_LIMIT).sum())
        self.count_over_f32 += int((finite > F32_EXP_LIMIT).sum())
        self.near_f16 += int((np.abs(finite - F16_EXP_LIMIT) <= NEAR_MARGIN).sum())
        self.near_f32 += int((np.abs(finite - F32_EXP_LIMIT) <= NEAR_MARGIN).sum())

    def record_gap(self, m_seed, exact_m):
        """src/vfa.py:129-135."""
        gap = m_seed - exact_m
        self.gap = gap
        self.calibration_gap = gap_summary([gap])


def gap_summary(gaps):
    """The calibration_gap dict (src/vfa.py:131-135) over the concatenated per-row gaps."""
    gap = np.concatenate([np.asarray(g, dtype=np.float64) for g in gaps])
    return {"min": float(gap.min()), "max": float(gap.max()), "mean": float(gap.mean()),
            "frac_below": float((gap < 0).mean())}


def exact_rowmax_global(q, k, scale, causal, rows=None):
    """src/reference.py:55-63, 105-111: per-row maximum over all unmasked scaled scores,
    (q @ k.T) * scale with the entrywise causal mask. rows: optional index array of query rows
    (the full-matrix product is then restricted to them; used for large problems)."""
    qq = q if rows is None else q[rows]
    s = (qq @ k.T) * scale
    if causal:
        r = np.arange(q.shape[0]) if rows is None else np.asarray(rows)
        cols = np.arange(k.shape[0])
        s[cols[None, :] > r[:, None]] = NEG_INF
    m = s.max(axis=1)
    if np.isneginf(m).any():
        raise FullyMaskedRow(int(np.argmax(np.isneginf(m))))
    return m


@dataclass
class HeadResult:
    out: np.ndarray
    lse: np.ndarray
    visited: int = 0
    skipped: int = 0
    special: int = 0
    frozen: int = 0
    monitor: Monitor = field(default_factory=Monitor)
    # per q-block list of (block j, skipped?, margin) in visit order (VSA only)
    decisions: list = field(default_factory=list)
    error: Exception | None = None
    elided: int = 0       # BLASST-FA4: processed blocks whose rescale was elided
    rows_masked: int = 0  # BLASST rowskip: suppressed row slots (skipped blocks count all rows)
    # StateTrace stabilization position per row (src/analysis.py:39-78): the block of the
    # first visit whose running-max snapshot equals the final max = the last visit that
    # raised it (the first visit if none did)
    stab: np.ndarray | None = None


VARIANTS = ("fa", "vfa", "vsa", "blasst", "blasst_fa4", "blasst_rowskip")
BLASST_VARIANTS = ("blasst", "blasst_fa4", "blasst_rowskip")


def forward_head(q, k, v, *, variant="vfa", causal=False, q_block=128, k_block=128,
                 scale=None, kind="sabsmax", qkind="row_wise", reorder=True,
                 use_m_init=True, tc1=None, n_sink=1, n_local=1, lam=None, tau=0.0,
                 order="sequential", raise_errors=True, record_decisions=False,
                 q_blocks=None, monitor=False) -> HeadResult:
    """One head of fa_forward (src/fa.py:28-61), vfa_forward (src/vfa.py:156-223),
    vsa_forward (src/sparse.py:256-329) or the BLASST family -- blasst_forward (order
    'sequential' | 'sink_local', src/sparse.py:112-152), blasst_fa4_forward (tau rescale
    elision, :155-203), blasst_rowskip_forward (row-granular, :206-253) -- float64,
    returning O, LSE and visit statistics.

    q_blocks: optional iterable of 1-based query blocks to compute (the others are left
    NaN); used to time bounded samples of large problems. Query blocks are independent
    (SPEC.md:212), so a sampled block is computed exactly as in the full pass.
    monitor: also record the calibration gap (src/vfa.py:217-221, src/sparse.py:324-327) when
    the m-init seeds are in use; the argument statistics are recorded on every call, like the
    reference.
    """
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    q = np.ascontiguousarray(q, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    nq, d = q.shape
    nk = k.shape[0]
    qb, kb = q_block, k_block
    if nq % qb or nk % kb:
        raise ValueError("sequence lengths must be divisible by the block sizes")
    if causal and nq != nk:
        raise ValueError("causal masking requires N_q == N_k")
    if scale is None:
        scale = 1.0 / np.sqrt(d)  # src/reference.py:45-46
    if variant == "fa":
        reorder, use_m_init, n_sink = False, False, 0
    if variant == "vsa":
        reorder, use_m_init = True, True  # src/sparse.py:288-290
    if variant in BLASST_VARIANTS:
        if variant == "blasst" and order not in ("sequential", "sink_local"):
            raise ValueError(f"unknown order {order!r}")  # src/sparse.py:121-122
        # m0 = -inf, every visited block takes the exact update; only blasst may reorder
        reorder = variant == "blasst" and order == "sink_local"
        use_m_init, n_sink, n_local = False, 1, 1
    skipping = variant in ("vsa", "blasst", "blasst_fa4", "blasst_rowskip")
    ln_lam = NEG_INF if (not skipping or lam is None) else math.log(lam)
    if skipping and lam is not None and not (0.0 < lam <= 1.0):
        raise ValueError(f"lambda must be in (0, 1], got {lam}")
    if tau < 0:
        raise ValueError(f"tau must be >= 0, got {tau}")  # src/sparse.py:52-53
    tau_ln2 = tau * math.log(2.0)
    t_r, t_c = nq // qb, nk // kb
    out = np.full((nq, d), np.nan)
    lse = np.full(nq, np.nan)
    res = HeadResult(out=out, lse=lse, stab=np.zeros(nq, dtype=np.int64))
    kreprs = precompute_kreprs(k, kb, kind, tc1) if use_m_init else None
    seeds = np.full(nq, np.nan) if (monitor and use_m_init) else None
    blocks_done = []

    for i in (range(1, t_r + 1) if q_blocks is None else q_blocks):
        blocks_done.append(i)
        vmax = visible_key_blocks(i, qb, kb, t_c, causal)
        local = local_key_block(i, qb, kb, t_c)
        if variant in ("fa", "blasst", "blasst_fa4", "blasst_rowskip"):
            if reorder:  # blasst order='sink_local': the VFA visit order, every block exact
                visit, _ = build_schedule(i, vmax, local, True, n_sink, n_local)
            else:
                visit = tuple(range(1, vmax + 1))
            special = frozenset(range(1, vmax + 1))
        else:
            visit, special = build_schedule(i, vmax, local, reorder, n_sink, n_local)
        qi = q[(i - 1) * qb: i * qb]
        if use_m_init:
            m = m_init(qi, kreprs[: min(vmax, len(kreprs))], scale, qkind)
        else:
            m = np.full(qb, NEG_INF)
        if seeds is not None:
            seeds[(i - 1) * qb: i * qb] = m
        l = np.zeros(qb)
        o = np.zeros((qb, d))
        dec = []
        stab = np.full(qb, visit[0], dtype=np.int64)
        for j in visit:
            s = tile_scores(q, k, scale, causal, i, j, qb, kb)
            v_j = v[(j - 1) * kb: j * kb]
            res.visited += 1
            need_max = (j in special) or variant == "vsa"
            if need_max:
                m_tilde = s.max(axis=1)
                m_new = np.maximum(m, m_tilde)
            if variant == "blasst_rowskip":  # src/sparse.py:223-249
                with np.errstate(invalid="ignore"):
                    keep = (m_tilde - m_new) >= ln_lam
                if ln_lam == NEG_INF:
                    keep = np.ones(qb, dtype=bool)
                if record_decisions:
                    dec.append((j, not keep.any(), _skip_margin(m_tilde, m_new, ln_lam)))
                if not keep.any():
                    res.skipped += 1
                    res.rows_masked += qb
                    continue
                f = np.where(keep, _rescale_factor(m, m_new), 1.0)
                s_kept = np.where(keep[:, None], s, NEG_INF)
                p_t = np.exp(_exp_args(s_kept, m_new))
                l = f * l + _rowsum(p_t)
                o = f[:, None] * o + p_t @ v_j
                m_next = np.where(keep, m_new, m)
                stab[m_next > m] = j
                m = m_next
                res.special += 1
                res.rows_masked += qb - int(keep.sum())
                continue
            if skipping:
                skip = _tile_skippable(m_tilde, m_new, ln_lam)
                if record_decisions:
                    dec.append((j, skip, _skip_margin(m_tilde, m_new, ln_lam)))
                if skip:
                    res.skipped += 1
                    continue
            if variant == "blasst_fa4":  # src/sparse.py:185-199
                prev_finite = not np.isneginf(m).any()
                if prev_finite and float(np.max(m_new - m)) <= tau_ln2:
                    args = _exp_args(s, m)
                    with np.errstate(over="ignore"):
                        p_t = np.exp(args)
                    l = l + _rowsum(p_t)
                    o = o + p_t @ v_j
                    res.frozen += 1
                    res.elided += 1
                    continue
            if j in special:
                args = _exp_args(s, m_new)
                res.monitor.record(args)
                p_t = np.exp(args)
                f = _rescale_factor(m, m_new)
                l = f * l + _rowsum(p_t)
                o = f[:, None] * o + p_t @ v_j
                stab[m_new > m] = j
                m = m_new
                res.special += 1
            else:
                args = _exp_args(s, m)
                res.monitor.record(args)
                with np.errstate(over="ignore"):
                    p_t = np.exp(args)
                l = l + _rowsum(p_t)
                o = o + p_t @ v_j
                res.frozen += 1
        if record_decisions:
            res.decisions.append(dec)
        res.stab[(i - 1) * qb: i * qb] = stab
        zero = l == 0.0  # src/core.py:101-109
        if zero.any():
            row = int(np.argmax(zero))
            err = (FullyMaskedRow if np.isneginf(m[row]) else NormalizerUnderflow)((i - 1) * qb + row)
            if raise_errors:
                raise err
            if res.error is None:
                res.error = err
        with np.errstate(divide="ignore", invalid="ignore"):
            out[(i - 1) * qb: i * qb] = o / l[:, None]
            lse[(i - 1) * qb: i * qb] = m + np.log(l)
    if seeds is not None:
        rows = None if q_blocks is None else np.concatenate(
            [np.arange((i - 1) * qb, i * qb) for i in blocks_done])
        exact = exact_rowmax_global(q, k, scale, causal, rows)
        res.monitor.record_gap(seeds if rows is None else seeds[rows], exact)
    return res


def forward(q, k, v, **kw):
    """Batched [B, Hq, L, d] / [B, Hkv, L, d] forward with GQA; returns (O, LSE, stats).

    O: float64 [B, Hq, Lq, d]; LSE: float64 [B, Hq, Lq]; stats: dict of summed counts.
    """
    q = np.asarray(q)
    k = np.asarray(k)
    v = np.asarray(v)
    if q.ndim == 2:
        r = forward_head(q, k, v, **kw)
        return r.out, r.lse, _stats([r])
    b, hq, lq, d = q.shape
    hkv = k.shape[1]
    if hq % hkv:
        raise ValueError("Hq must be a multiple of Hkv")
    grp = hq // hkv
    out = np.empty((b, hq, lq, d))
    lse = np.empty((b, hq, lq))
    results = []
    for bi in range(b):
        for h in range(hq):
            r = forward_head(q[bi, h], k[bi, h // grp], v[bi, h // grp], **kw)
            out[bi, h] = r.out
            lse[bi, h] = r.lse
            results.append(r)
    return out, lse, _stats(results)


def _stats(results):
    st = {"visited": 0, "skipped": 0, "special": 0, "frozen": 0, "elided": 0, "rows_masked": 0,
          "count_over_f16": 0, "count_over_f32": 0, "near_f16": 0, "near_f32": 0,
          "exp_arg_max": NEG_INF, "calibration_gap": None}
    gaps = [r.monitor.gap for r in results if r.monitor.gap is not None]
    if gaps:
        st["calibration_gap"] = gap_summary(gaps)
    for r in results:
        st["near_f16"] += r.monitor.near_f16
        st["near_f32"] += r.monitor.near_f32
        st["elided"] += r.elided
        st["rows_masked"] += r.rows_masked
        st["visited"] += r.visited
        st["skipped"] += r.skipped
        st["special"] += r.special
        st["frozen"] += r.frozen
        st["count_over_f16"] += r.monitor.count_over_f16
        st["count_over_f32"] += r.monitor.count_over_f32
        st["exp_arg_max"] = max(st["exp_arg_max"], r.monitor.exp_arg_max)
    return st


def causal_flops(b, hq, lq, d):
    """Algorithmic FLOPs of a causal forward, 4*B*Hq*L^2*d/2."""
    return 4.0 * b * hq * lq * lq * d / 2.0


def max_rel_err(a, b):
    """tests/conftest.py:42-46: max over rows of ||a_r - b_r||_inf / ||b_r||_inf."""
    a = np.asarray(a, dtype=np.float64).reshape(-1, np.shape(a)[-1])
    b = np.asarray(b, dtype=np.float64).reshape(-1, np.shape(b)[-1])
    diff = np.abs(a - b).max(axis=1)
    denom = np.maximum(np.abs(b).max(axis=1), np.finfo(np.float64).tiny)
    return float((diff / denom).max())
