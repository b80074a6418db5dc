"""Drop-in host API mirroring the reference's attention entry points.

Reference (src/X.py = /root/reference/pkg/src/vfa_lab/X.py):
  BlockSpec                      src/tensor.py:19-52
  AttentionProblem               src/reference.py:20-54
  SkipConfig / SkipStats         src/sparse.py:41-96
  OpCounters charges             src/counters.py:59-100
  fa_forward                     src/fa.py:28-61
  vfa_forward                    src/vfa.py:156-223
  vsa_forward                    src/sparse.py:256-329
  precompute_kreprs              src/vfa.py:79-88
  FullyMaskedRowError / NormalizerUnderflowError   src/errors.py:4-17

Same names, keyword arguments, validation errors and numerical exceptions; the
compute runs in libvfa_b200.so (hand-written sm_100a kernels) on bf16 CUDA
tensors. Differences that follow from running on the GPU: O is returned as a bf16
torch tensor on the device (shape of q), the LSE is returned as well (`.lse`),
`trace` is a DeviceTrace (the per-row stabilization positions the reference's
StateTrace feeds into stabilization_positions, recorded by the kernel instead of per-visit
m snapshots), and the OverflowMonitor statistics come from device counters when
monitor=True.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, fields

import numpy as np
import torch

from . import _lib

NEG_INF = float("-inf")
LN2 = math.log(2.0)


# ----------------------------------------------------------------------------- errors
class FullyMaskedRowError(ValueError):
    """A query row has every score masked; its softmax is undefined (src/errors.py:4-9)."""

    def __init__(self, row: int):
        self.row = row
        super().__init__(f"query row {row} is fully masked; cannot normalize")


class NormalizerUnderflowError(ArithmeticError):
    """A softmax normalizer underflowed to zero at finalization (src/errors.py:12-17)."""

    def __init__(self, row: int):
        self.row = row
        super().__init__(f"normalizer underflow at query row {row}")


class KernelError(RuntimeError):
    """CUDA launch/runtime failure inside libvfa_b200 (C-ABI code 5)."""


# ----------------------------------------------------------------------------- problem
@dataclass(frozen=True)
class BlockSpec:
    """Tile geometry (src/tensor.py:19-52): lengths must divide by the block sizes."""

    seq_len_q: int
    seq_len_k: int
    head_dim: int
    q_block: int = 128
    k_block: int = 128

    def __post_init__(self):
        for name in ("seq_len_q", "seq_len_k", "head_dim", "q_block", "k_block"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")
        if self.seq_len_q % self.q_block != 0:
            raise ValueError(f"seq_len_q={self.seq_len_q} not divisible by q_block={self.q_block}")
        if self.seq_len_k % self.k_block != 0:
            raise ValueError(f"seq_len_k={self.seq_len_k} not divisible by k_block={self.k_block}")

    @property
    def t_r(self) -> int:
        return self.seq_len_q // self.q_block

    @property
    def t_c(self) -> int:
        return self.seq_len_k // self.k_block


def _as_device_bf16(x, device):
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if not isinstance(x, torch.Tensor):
        raise TypeError("q, k, v must be torch tensors or numpy arrays")
    if x.dtype != torch.bfloat16 or x.device.type != "cuda":
        x = x.to(device=device, dtype=torch.bfloat16)
    return x


@dataclass
class AttentionProblem:
    """One attention invocation (src/reference.py:20-54).

    q: [Nq, d] or [B, Hq, Nq, d]; k, v: [Nk, d] or [B, Hkv, Nk, d] (Hq % Hkv == 0, GQA).
    Tensors are moved to the GPU as bf16 if they are not already.
    """

    q: object
    k: object
    v: object
    blocks: BlockSpec | None = None
    scale: float | None = None
    causal: bool = False

    def __post_init__(self):
        # validate shapes first (src/reference.py:31-46), then move to the GPU
        qs, ks, vs = (tuple(np.shape(x)) if not isinstance(x, torch.Tensor) else tuple(x.shape)
                      for x in (self.q, self.k, self.v))
        if len(qs) not in (2, 4) or len(ks) != len(qs) or len(vs) != len(qs):
            raise ValueError("q, k, v must all be 2-D [N, d] or all 4-D [B, H, N, d]")
        n_q, d = qs[-2], qs[-1]
        if ks[-1] != d or vs[-1] != d:
            raise ValueError("Q, K, V must share the head dimension")
        if ks != vs:
            raise ValueError("K and V must have the same number of rows")
        if len(qs) == 4:
            if qs[0] != ks[0]:
                raise ValueError("Q and K/V batch sizes differ")
            if qs[1] % ks[1]:
                raise ValueError("query heads must be a multiple of key/value heads")
        n_k = ks[-2]
        if self.blocks is None:
            self.blocks = BlockSpec(n_q, n_k, d, 128, 128)
        if (n_q, n_k, d) != (self.blocks.seq_len_q, self.blocks.seq_len_k, self.blocks.head_dim):
            raise ValueError("tensor shapes do not match the block spec")
        if self.causal and n_q != n_k:
            raise ValueError("causal masking requires N_q == N_k")
        if self.scale is None:
            self.scale = 1.0 / math.sqrt(d)
        dev = None
        for x in (self.q, self.k, self.v):
            if isinstance(x, torch.Tensor) and x.device.type == "cuda":
                dev = x.device
        dev = dev or torch.device("cuda", torch.cuda.current_device() if torch.cuda.is_available() else 0)
        self.q = _as_device_bf16(self.q, dev)
        self.k = _as_device_bf16(self.k, dev)
        self.v = _as_device_bf16(self.v, dev)

    @property
    def t_r(self) -> int:
        return self.blocks.t_r

    @property
    def t_c(self) -> int:
        return self.blocks.t_c


# ----------------------------------------------------------------------------- skip config / stats
@dataclass(frozen=True)
class SkipConfig:
    """Skip thresholds (src/sparse.py:41-59). lam=None disables skipping."""

    lam: float | None
    tau: float = 0.0
    granularity: str = "block"

    def __post_init__(self):
        if self.lam is not None and not (0.0 < self.lam <= 1.0):
            raise ValueError(f"lambda must be in (0, 1], got {self.lam}")
        if self.tau < 0:
            raise ValueError(f"tau must be >= 0, got {self.tau}")
        if self.granularity not in ("block", "row"):
            raise ValueError(f"granularity must be 'block' or 'row', got {self.granularity!r}")

    @property
    def ln_lambda(self) -> float:
        return NEG_INF if self.lam is None else math.log(self.lam)


@dataclass
class SkipStats:
    """src/sparse.py:62-96 (the fields the block-granular VSA pass fills)."""

    blocks_visited: int = 0
    blocks_skipped: int = 0
    rows_masked: int = 0
    row_slots: int = 0
    rescales_elided: int = 0
    blocks_processed: int = 0
    processed_special: int = 0
    processed_frozen: int = 0

    @property
    def block_sparsity(self) -> float:
        return self.blocks_skipped / self.blocks_visited if self.blocks_visited else 0.0

    @property
    def row_sparsity(self) -> float:
        return self.rows_masked / self.row_slots if self.row_slots else 0.0

    @property
    def rescale_skip_rate(self) -> float:
        return self.rescales_elided / self.blocks_processed if self.blocks_processed else 0.0

    def as_dict(self) -> dict:
        """src/sparse.py:84-96 (the reference reports these fields)."""
        d = {f.name: getattr(self, f.name) for f in fields(self) if f.name not in ("processed_special",
                                                                                 "processed_frozen")}
        d["block_sparsity"] = self.block_sparsity
        d["row_sparsity"] = self.row_sparsity
        d["rescale_skip_rate"] = self.rescale_skip_rate
        return d


@dataclass
class OpCounters:
    """Element-level op accounting (src/counters.py:14-43), charged per block class
    from the device's per-class block counts, so it is integer-equal to the
    reference's instrumented counters whenever the visit statistics agree."""

    mul_scale: int = 0
    max_rowreduce: int = 0
    max_running: int = 0
    sub_broadcast: int = 0
    exp_evals: int = 0
    sum_rowreduce: int = 0
    mad_l: int = 0
    rescale_mul_l: int = 0
    rescale_mul_O: int = 0
    tensor_macs: int = 0
    rowmax_reductions: int = 0
    rescale_events: int = 0
    blocks_processed: int = 0
    blocks_skipped: int = 0
    rescales_elided: int = 0
    rows_masked: int = 0

    def as_dict(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}

    def charge(self, full: int, frozen: int, skipped: int, q: int, k: int, d: int, frozen_rowmax: bool):
        """n * charge_full_block + m * charge_frozen_block + s * charge_skipped_block."""
        qk = q * k
        self.mul_scale += (full + frozen + skipped) * qk
        self.max_rowreduce += (full + skipped + (frozen if frozen_rowmax else 0)) * qk
        self.max_running += (full + skipped + (frozen if frozen_rowmax else 0)) * q
        self.sub_broadcast += (full + frozen) * qk
        self.exp_evals += full * (qk + q) + frozen * qk
        self.sum_rowreduce += (full + frozen) * qk
        self.mad_l += (full + frozen) * q
        self.rescale_mul_l += full * q
        self.rescale_mul_O += full * q * d
        self.tensor_macs += (full + frozen) * 2 * qk * d + skipped * qk * d
        self.rowmax_reductions += full + skipped + (frozen if frozen_rowmax else 0)
        self.rescale_events += full
        self.blocks_processed += full + frozen
        self.blocks_skipped += skipped

    @classmethod
    def from_stats(cls, variant: str, st: dict, q: int, k: int, d: int) -> "OpCounters":
        """Counters of a whole pass from its per-class block counts (device stats or oracle
        results: visited / skipped / special / frozen / elided / rows_masked), charged
        exactly as the reference variant charges each block."""
        c = cls()
        if variant == "blasst_rowskip":
            skipped_rows = st["skipped"] * q
            kept = st["special"] * q - (st["rows_masked"] - skipped_rows)
            c.charge(0, 0, st["skipped"], q, k, d, False)
            c.charge_rowskip(st["special"], kept, q, k, d)
            c.rows_masked += skipped_rows  # src/sparse.py:232-233
        elif variant == "blasst_fa4":
            c.charge(st["special"], 0, st["skipped"], q, k, d, False)
            c.charge_elided(st["elided"], q, k, d)
        else:
            c.charge(st["special"], st["frozen"], st["skipped"], q, k, d, variant == "vsa")
        return c

    def charge_elided(self, n: int, q: int, k: int, d: int):
        """n * charge_elided_block (src/counters.py:102-114)."""
        qk = q * k
        self.mul_scale += n * qk
        self.max_rowreduce += n * qk
        self.max_running += n * q
        self.sub_broadcast += n * qk
        self.exp_evals += n * qk
        self.sum_rowreduce += n * qk
        self.mad_l += n * q
        self.tensor_macs += n * 2 * qk * d
        self.rowmax_reductions += n
        self.rescales_elided += n
        self.blocks_processed += n

    def charge_rowskip(self, n: int, kept: int, q: int, k: int, d: int):
        """Sum of charge_rowskip_block (src/counters.py:116-131) over n processed blocks that
        kept `kept` rows in total (the charge is linear in kept)."""
        qk = q * k
        self.mul_scale += n * qk
        self.max_rowreduce += n * qk
        self.max_running += n * q
        self.sub_broadcast += kept * k
        self.exp_evals += kept * k + kept
        self.sum_rowreduce += kept * k
        self.mad_l += n * q
        self.rescale_mul_l += kept
        self.rescale_mul_O += kept * d
        self.tensor_macs += n * 2 * qk * d
        self.rowmax_reductions += n
        self.rescale_events += n
        self.rows_masked += n * q - kept
        self.blocks_processed += n


@dataclass
class OverflowMonitor:
    """src/vfa.py:109-135: exp arguments > ln 65504 and > 88.7228 counted on the device, the
    largest argument, and the calibration gap (m seed - exact global row max: min / max / mean /
    frac_below) from the device's seeds and exact row maxima (monitor=True)."""

    exp_arg_max: float = NEG_INF
    count_over_f16: int = 0
    count_over_f32: int = 0
    calibration_gap: dict | None = None


class ForwardResult(tuple):
    """Tuple with the reference's arity plus `.lse` (fp32, [..., Nq]) and `.stats`."""

    lse: torch.Tensor
    stats: dict

    def __new__(cls, items, lse, stats):
        obj = super().__new__(cls, items)
        obj.lse = lse
        obj.stats = stats
        return obj


# ----------------------------------------------------------------------------- core launcher
def _strides(x):
    s = x.stride()
    if x.stride(-1) != 1:
        raise ValueError("the head dimension must be contiguous")
    return (s[0], s[1], s[2])


def _params(q, k, v, o, *, variant, causal, q_block, k_block, scale, kind, qkind, reorder,
            use_m_init, tc1, n_sink, n_local, lam, monitor, softmax_split=0, tau=0.0, cta_pair=0):
    if kind not in _lib.KEY_REPRS:
        raise ValueError(f"unknown key representation {kind!r}")
    if qkind not in _lib.QUERY_REPRS:
        raise ValueError(f"unknown query representation {qkind!r}")
    p = _lib.VfaParams()
    p.batch, p.heads_q, p.seq_q, p.head_dim = q.shape
    p.heads_kv, p.seq_k = k.shape[1], k.shape[2]
    p.q_stride[:] = _strides(q)
    p.k_stride[:] = _strides(k)
    p.v_stride[:] = _strides(v)
    p.o_stride[:] = _strides(o)
    if scale is not None and not (math.isfinite(scale) and scale > 0):
        # the kernels fold the scale into exp2 after the row max: a positive finite scale keeps
        # max(s) * scale == max(s * scale); None (0.0 across the C ABI) means 1/sqrt(d)
        raise ValueError(f"scale must be a positive finite number, got {scale}")
    p.scale = float(scale) if scale is not None else 0.0
    p.causal = int(bool(causal))
    p.q_block, p.k_block = int(q_block), int(k_block)
    p.variant = _lib.VARIANTS[variant]
    p.kind = _lib.KEY_REPRS.index(kind)
    p.qkind = _lib.QUERY_REPRS.index(qkind)
    p.reorder = int(bool(reorder))
    p.use_m_init = int(bool(use_m_init))
    p.tc1 = 0 if tc1 is None else int(tc1)
    p.n_sink, p.n_local = int(n_sink), int(n_local)
    p.monitor = int(bool(monitor))
    p.lam = float(lam) if lam is not None else 0.0
    p.tau = float(tau)
    p.softmax_split = int(softmax_split)
    p.cta_pair = int(cta_pair)
    return p


def _check_shapes(q, k, v):
    """The AttentionProblem checks (src/reference.py:31-46) on [B, H, N, d] tensors: the C ABI
    takes batch and head_dim from q and the key length from k, so a mismatch must be caught
    here (it would otherwise index past the end of k / v)."""
    if tuple(k.shape) != tuple(v.shape):
        raise ValueError("K and V must have the same shape")
    if k.shape[0] != q.shape[0]:
        raise ValueError("Q and K/V batch sizes differ")
    if k.shape[3] != q.shape[3]:
        raise ValueError("Q, K, V must share the head dimension")
    if q.shape[1] % k.shape[1]:
        raise ValueError("query heads must be a multiple of key/value heads")


def _check_outputs(q, out, lse, dev):
    if not isinstance(out, torch.Tensor) or out.dtype != torch.bfloat16 or out.device != dev:
        raise ValueError("out must be a bf16 tensor on q's device")
    if tuple(out.shape) != tuple(q.shape) or out.stride(-1) != 1:
        raise ValueError(f"out must have q's shape {tuple(q.shape)} with a contiguous head dimension")
    if not isinstance(lse, torch.Tensor) or lse.dtype != torch.float32 or lse.device != dev:
        raise ValueError("lse must be a float32 tensor on q's device")
    if tuple(lse.shape) != tuple(q.shape[:3]) or not lse.is_contiguous():
        raise ValueError(f"lse must be a contiguous float32 tensor of shape {tuple(q.shape[:3])}")


def _raise_for(rc):
    msg = _lib.last_error()
    if rc in (_lib.VFA_ERR_CONFIG, _lib.VFA_ERR_DATA):
        raise ValueError(msg)
    raise KernelError(f"libvfa_b200 error {rc}: {msg}")


def attention_forward(q, k, v, *, variant="vfa", causal=False, q_block=128, k_block=128, scale=None,
                      kind="sabsmax", qkind="row_wise", reorder=True, use_m_init=True, tc1=None,
                      n_sink=1, n_local=1, lam=None, tau=0.0, monitor=False, out=None, lse=None,
                      check=True, skip_trace=False, stream=None, workspace=None,
                      krepr_precomputed=False, softmax_split=0, stab_trace=False, cta_pair=0,
                      state_trace=False):
    """Launch the B200 forward on bf16 CUDA tensors [B, Hq, Lq, d] / [B, Hkv, Lk, d].

    Returns (out, lse, info) with info = {"stats": int64 device tensor | dict,
    "status": uint32 device tensor, "skip_trace": uint8 device tensor | None}.
    With check=True the status word is read back (one device sync) and
    FullyMaskedRowError / NormalizerUnderflowError raised like src/core.py:101-109.
    workspace: optional uint8 device buffer (>= vfa_workspace_bytes) holding the key-block
    representations; with krepr_precomputed=True they are reused instead of recomputed.
    variant: fa | vfa | vsa | blasst | blasst_fa4 | blasst_rowskip. reorder selects the
    sink/local-first visit order (VFA / VSA; for blasst it is order='sink_local', so pass
    reorder=False for the reference's default sequential blasst). lam: skip threshold of the
    skipping variants; tau: blasst_fa4 rescale-elision threshold (SkipConfig.tau).
    stab_trace: also return info["stab_block"], int32 [B, Hq, Lq]: per row the key block after
    whose visit the running max held its final value (the StateTrace stabilization position,
    src/analysis.py:39-78), see DeviceTrace / stabilization_positions.
    state_trace: also return info["m_trace"], float32 [B, Hq, Lq, T_c]: the reference's StateTrace
    snapshots (src/core.py:35-54) -- per row and visit position (schedule order) the running max
    after the visit, natural units; NaN past the row's visible blocks (a debug output).
    cta_pair: 0 (default: off), 1 (one CTA per unit) or 2 (CTA pairs sharing each K/V tile
    through M = 256 tcgen05 MMAs: two query tiles per CTA for GQA groups divisible by 4, one for
    other even groups; d = 128, q_block = 128; falls back to single CTAs elsewhere).
    softmax_split: 0 (per-variant default), 1, 2 or 4 threads per row of a query tile (a layout
    choice: results are within tolerance of each other, bitwise-stable for a fixed split).
    """
    if variant not in _lib.VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    if variant not in ("fa", "vfa") and lam is not None and not (0.0 < lam <= 1.0):
        raise ValueError(f"lambda must be in (0, 1], got {lam}")
    if not tau >= 0:
        raise ValueError(f"tau must be >= 0, got {tau}")
    if all(isinstance(x, torch.Tensor) and x.device.type == "cpu" for x in (q, k, v)):
        if skip_trace or stab_trace or state_trace or krepr_precomputed or workspace is not None:
            raise ValueError("skip_trace / stab_trace / state_trace / krepr_precomputed / workspace need "
                             "device-resident inputs")
        return attention_forward_host(q, k, v, variant=variant, causal=causal, q_block=q_block,
                                      k_block=k_block, scale=scale, kind=kind, qkind=qkind,
                                      reorder=reorder, use_m_init=use_m_init, tc1=tc1, n_sink=n_sink,
                                      n_local=n_local, lam=lam, tau=tau, monitor=monitor, out=out, lse=lse,
                                      check=check, stream=stream, softmax_split=softmax_split,
                                      cta_pair=cta_pair)
    lib = _lib.load()
    for name, x in (("q", q), ("k", k), ("v", v)):
        if not isinstance(x, torch.Tensor) or x.dtype != torch.bfloat16 or x.device.type != "cuda":
            raise TypeError(f"{name} must be a bf16 CUDA tensor")
        if x.dim() != 4:
            raise ValueError(f"{name} must be 4-D [B, H, N, d]")
    _check_shapes(q, k, v)
    dev = q.device
    if k.device != dev or v.device != dev:
        raise ValueError("q, k and v must be on the same device")
    if out is None:
        out = torch.empty(q.shape, dtype=torch.bfloat16, device=dev)
    if lse is None:
        lse = torch.empty(q.shape[:3], dtype=torch.float32, device=dev)
    _check_outputs(q, out, lse, dev)
    p = _params(q, k, v, out, variant=variant, causal=causal, q_block=q_block, k_block=k_block,
                scale=scale, kind=kind, qkind=qkind, reorder=reorder, use_m_init=use_m_init,
                tc1=tc1, n_sink=n_sink, n_local=n_local, lam=lam, monitor=monitor,
                softmax_split=softmax_split, tau=tau, cta_pair=cta_pair)
    rc = lib.vfa_check_params(ctypes.byref(p))
    if rc:
        _raise_for(rc)
    p.krepr_precomputed = int(bool(krepr_precomputed))
    ws_bytes = int(lib.vfa_workspace_bytes(ctypes.byref(p)))
    if workspace is None:
        if krepr_precomputed:
            raise ValueError("krepr_precomputed needs the workspace that holds the representations")
        ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    else:
        if workspace.numel() < ws_bytes:
            raise ValueError(f"workspace too small: {workspace.numel()} < {ws_bytes}")
        ws = workspace
    stats = torch.empty(_lib.STAT_COUNT, dtype=torch.int64, device=dev)
    status = torch.empty(_lib.STATUS_COUNT, dtype=torch.int32, device=dev)
    trace = None
    if skip_trace:
        trace = torch.empty((q.shape[0], q.shape[1], q.shape[2] // q_block, k.shape[2] // k_block),
                            dtype=torch.uint8, device=dev)
    stab = torch.empty(q.shape[:3], dtype=torch.int32, device=dev) if stab_trace else None
    st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    m_trace = None
    with torch.cuda.device(dev):
        if state_trace:
            if skip_trace:
                raise ValueError("state_trace and skip_trace are separate debug runs")
            m_trace = torch.full((*q.shape[:3], k.shape[2] // k_block), float("nan"), dtype=torch.float32,
                                 device=dev)
            rc = lib.vfa_fwd_state_trace(ctypes.byref(p), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                         out.data_ptr(), lse.data_ptr(), ws.data_ptr(), ws_bytes,
                                         stats.data_ptr(), status.data_ptr(),
                                         stab.data_ptr() if stab is not None else None, m_trace.data_ptr(),
                                         ctypes.c_void_p(st))
        else:
            rc = lib.vfa_fwd(ctypes.byref(p), q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                             lse.data_ptr(), ws.data_ptr(), ws_bytes, stats.data_ptr(), status.data_ptr(),
                             trace.data_ptr() if trace is not None else None,
                             stab.data_ptr() if stab is not None else None, ctypes.c_void_p(st))
    if rc:
        _raise_for(rc)
    info = {"stats": stats, "status": status, "skip_trace": trace, "workspace": ws, "stab_block": stab,
            "m_trace": m_trace}
    if check:
        flags = int(status[_lib.STATUS_FLAGS].item())
        if flags & 2 and not flags & 1 and variant == "vfa" and use_m_init:
            # fp32 normalizer underflow with a finite frozen max: recompute those rows exactly
            # (or raise like the float64 reference when its own exp underflows too)
            with torch.cuda.device(dev):
                _rebase_underflow_rows(lib, p, q, k, v, out, lse, ws, ws_bytes, st, status)
            info["rebased_rows"] = True
            return out, lse, info
        check_status(status)
    return out, lse, info


# np.exp(x) == 0 in float64 for x below this (src/core.py:101-109: the reference's l underflows)
F64_EXP_UNDERFLOW = -745.1332191019412


def _rebase_underflow_rows(lib, p, q, k, v, out, lse, ws, ws_bytes, st, first_status):
    """Recovery of rows whose fp32 normalizer underflowed (include/vfa_b200.h, vfa_fwd_rebased).

    VFA freezes the running max at its m-init seed; when the seed exceeds every score of a row by
    more than fp32's exp range (~87 nats) each exponential flushes to zero on the device, while
    the float64 reference (src/vfa.py:209-215, src/core.py:95-109) still normalizes the row. The
    kernel flags such rows (O = NaN, the frozen max in the LSE slot); here their exact row max is
    computed (q . k^T over the visible keys, fp32), and the forward re-runs with the per-row
    exponent rebase 2^(frozen - exact). Rows whose gap exceeds float64's exp range raise
    NormalizerUnderflowError like the reference."""
    flagged = torch.isnan(out[..., 0]) & torch.isfinite(lse)
    idx = flagged.nonzero()
    if idx.numel() == 0:  # (the kernel flags every such row; keep the first pass's error)
        check_status(first_status)
    B, Hq, Lq, d = q.shape
    group = Hq // k.shape[1]
    scale = p.scale if p.scale > 0 else 1.0 / math.sqrt(d)
    exact = torch.empty(idx.shape[0], dtype=torch.float32, device=q.device)
    lin = (idx[:, 0] * Hq + idx[:, 1]) * Lq + idx[:, 2]
    order = torch.argsort(lin)
    idx, lin = idx[order], lin[order]
    heads = torch.unique(idx[:, 0] * Hq + idx[:, 1]).tolist()
    for bh in heads:
        b, h = divmod(int(bh), Hq)
        sel = ((idx[:, 0] == b) & (idx[:, 1] == h)).nonzero().flatten()
        kk = k[b, h // group].float()
        for c0 in range(0, sel.numel(), 2048):
            rows_i = sel[c0:c0 + 2048]
            rows = idx[rows_i, 2]
            s = (q[b, h, rows].float() @ kk.T) * scale
            if p.causal:
                cols = torch.arange(kk.shape[0], device=q.device)
                s = s.masked_fill(cols[None, :] > rows[:, None], float("-inf"))
            exact[rows_i] = s.max(dim=1).values
    frozen = lse[idx[:, 0], idx[:, 1], idx[:, 2]]
    gap = frozen.double() - exact.double()
    dead = (-gap < F64_EXP_UNDERFLOW).nonzero()
    if dead.numel():
        raise NormalizerUnderflowError(int(lin[dead[0, 0]].item()))
    bias = torch.zeros(q.shape[:3], dtype=torch.float32, device=q.device)
    bias[idx[:, 0], idx[:, 1], idx[:, 2]] = (gap / LN2).float()
    stats = torch.empty(_lib.STAT_COUNT, dtype=torch.int64, device=q.device)
    status = torch.empty(_lib.STATUS_COUNT, dtype=torch.int32, device=q.device)
    p2 = _lib.VfaParams.from_buffer_copy(p)
    p2.krepr_precomputed = 1  # the representations of the first pass are still in `ws`
    rc = lib.vfa_fwd_rebased(ctypes.byref(p2), q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                             lse.data_ptr(), ws.data_ptr(), ws_bytes, stats.data_ptr(), status.data_ptr(),
                             bias.data_ptr(), ctypes.c_void_p(st))
    if rc:
        _raise_for(rc)
    check_status(status)


def attention_forward_host(q, k, v, *, variant="vfa", causal=False, q_block=128, k_block=128,
                           scale=None, kind="sabsmax", qkind="row_wise", reorder=True, use_m_init=True,
                           tc1=None, n_sink=1, n_local=1, lam=None, tau=0.0, monitor=False, out=None,
                           lse=None,
                           check=True, stream=None, device=None, chunk_kv_heads=1, chunk_q_heads=2,
                           softmax_split=0, cta_pair=0):
    """The forward on HOST tensors (bf16 [B, Hq, Lq, d] / [B, Hkv, Lk, d], contiguous;
    page-locked for full overlap) -> host (O bf16, LSE fp32, info), through the C ABI's
    vfa_fwd_host: chunks of `chunk_kv_heads` KV heads are copied in, computed and copied
    out on overlapping streams, so the PCIe transfers hide behind the attention kernels;
    each KV head's K/V is copied once and its query heads go in sub-chunks of chunk_q_heads
    (when chunk_kv_heads == 1 and it divides the GQA group; else whole groups).
    The result is in host memory when this returns (check=True) or once `stream` (default:
    the current stream of `device`) is synchronized (check=False)."""
    lib = _lib.load()
    for name, x in (("q", q), ("k", k), ("v", v)):
        if not isinstance(x, torch.Tensor) or x.dtype != torch.bfloat16 or x.device.type != "cpu":
            raise TypeError(f"{name} must be a bf16 CPU tensor")
        if x.dim() != 4:
            raise ValueError(f"{name} must be 4-D [B, H, N, d]")
        if not x.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
    _check_shapes(q, k, v)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    pin = q.is_pinned()
    if out is None:
        out = torch.empty(q.shape, dtype=torch.bfloat16, pin_memory=pin)
    if lse is None:
        lse = torch.empty(q.shape[:3], dtype=torch.float32, pin_memory=pin)
    for name, x, dt in (("out", out, torch.bfloat16), ("lse", lse, torch.float32)):
        if x.device.type != "cpu" or x.dtype != dt or not x.is_contiguous():
            raise ValueError(f"{name} must be a contiguous {dt} CPU tensor")
    if tuple(out.shape) != tuple(q.shape) or tuple(lse.shape) != tuple(q.shape[:3]):
        raise ValueError("out / lse shapes do not match q")
    p = _params(q, k, v, out, variant=variant, causal=causal, q_block=q_block, k_block=k_block,
                scale=scale, kind=kind, qkind=qkind, reorder=reorder, use_m_init=use_m_init,
                tc1=tc1, n_sink=n_sink, n_local=n_local, lam=lam, monitor=monitor,
                softmax_split=softmax_split, tau=tau, cta_pair=cta_pair)
    rc = lib.vfa_check_params(ctypes.byref(p))
    if rc:
        _raise_for(rc)
    group = q.shape[1] // k.shape[1]
    cq = int(chunk_q_heads) if (chunk_kv_heads == 1 and chunk_q_heads and group % chunk_q_heads == 0) else 0
    nbytes = int(lib.vfa_host_scratch_bytes(ctypes.byref(p), int(chunk_kv_heads), cq))
    if nbytes == 0:
        raise ValueError(f"chunk_kv_heads={chunk_kv_heads} must divide heads_kv={k.shape[1]}")
    with torch.cuda.device(dev):
        scratch = torch.empty(nbytes, dtype=torch.uint8, device=dev)
        stats = torch.empty(_lib.STAT_COUNT, dtype=torch.int64, device=dev)
        status = torch.empty(_lib.STATUS_COUNT, dtype=torch.int32, device=dev)
        st = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
        rc = lib.vfa_fwd_host(ctypes.byref(p), q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                              lse.data_ptr(), scratch.data_ptr(), nbytes, stats.data_ptr(),
                              status.data_ptr(), int(chunk_kv_heads), cq, ctypes.c_void_p(st))
    if rc:
        _raise_for(rc)
    info = {"stats": stats, "status": status, "skip_trace": None, "workspace": None}
    if check:
        flags = int(status[_lib.STATUS_FLAGS].item())  # synchronizes with the stream
        if flags & 2 and not flags & 1 and variant == "vfa" and use_m_init:
            # fp32 normalizer underflow: the (rare) recovery runs on device-resident copies
            o_d, l_d, info = attention_forward(
                q.to(dev), k.to(dev), v.to(dev), variant=variant, causal=causal, q_block=q_block,
                k_block=k_block, scale=scale, kind=kind, qkind=qkind, reorder=reorder,
                use_m_init=use_m_init, tc1=tc1, n_sink=n_sink, n_local=n_local, lam=lam, tau=tau,
                monitor=monitor, check=True, softmax_split=softmax_split, cta_pair=cta_pair)
            out.copy_(o_d.cpu())
            lse.copy_(l_d.cpu())
            return out, lse, info
        check_status(status)
        torch.cuda.synchronize(dev)
    return out, lse, info


def check_status(status: torch.Tensor):
    """Raise the reference's finalize errors from a device status word (src/core.py:101-109)."""
    s = status.cpu().numpy().view(np.uint32)
    flags = int(s[_lib.STATUS_FLAGS])
    if flags & 1:
        raise FullyMaskedRowError(int(s[_lib.STATUS_MASKED_ROW]))
    if flags & 2:
        raise NormalizerUnderflowError(int(s[_lib.STATUS_UNDERFLOW_ROW]))
    return flags


def stats_dict(info) -> dict:
    s = info["stats"].cpu().tolist()
    d = {"visited": s[_lib.STAT_VISITED], "skipped": s[_lib.STAT_SKIPPED],
         "special": s[_lib.STAT_SPECIAL], "frozen": s[_lib.STAT_FROZEN],
         "elided": s[_lib.STAT_ELIDED], "rows_masked": s[_lib.STAT_ROWS_MASKED],
         "count_over_f32": s[_lib.STAT_OVER_F32], "count_over_f16": s[_lib.STAT_OVER_F16],
         "nonfinite_rows": int(info["status"].cpu()[_lib.STATUS_NONFINITE_ROWS])}
    # monitor statistics (log2 units on the device -> natural units, src/vfa.py:109-135)
    amax = _lib.key_to_float(s[_lib.STAT_EXP_ARG_MAX])
    d["exp_arg_max"] = NEG_INF if math.isnan(amax) else amax * LN2
    rows = s[_lib.STAT_GAP_ROWS]
    if rows:
        gsum = np.array([s[_lib.STAT_GAP_SUM]], dtype=np.int64).view(np.float64)[0]
        d["calibration_gap"] = {"min": -_lib.key_to_float(s[_lib.STAT_GAP_NEG_MIN]) * LN2,
                                "max": _lib.key_to_float(s[_lib.STAT_GAP_MAX]) * LN2,
                                "mean": float(gsum) / rows * LN2,
                                "frac_below": s[_lib.STAT_GAP_BELOW] / rows}
    else:
        d["calibration_gap"] = None
    return d


# ----------------------------------------------------------------------------- reference-shaped entry points
def _run(p: AttentionProblem, variant, **kw):
    q, k, v = p.q, p.k, p.v
    two_d = q.dim() == 2
    if two_d:
        q, k, v = (x.view(1, 1, *x.shape) for x in (q, k, v))
    out, lse, info = attention_forward(q, k, v, variant=variant, causal=p.causal,
                                       q_block=p.blocks.q_block, k_block=p.blocks.k_block,
                                       scale=p.scale, **kw)
    st = stats_dict(info)
    if info.get("stab_block") is not None:
        st["stab_block"] = info["stab_block"].view(*p.q.shape[:-1]) if two_d else info["stab_block"]
    if info.get("m_trace") is not None:
        mt = info["m_trace"]
        st["m_trace"] = mt.view(*p.q.shape[:-1], mt.shape[-1]) if two_d else mt
    if two_d:
        out, lse = out.view(*p.q.shape), lse.view(p.q.shape[0])
    return out, lse, st


@dataclass
class DeviceTrace:
    """Device-side stand-in for the reference's StateTrace (src/core.py:35-54).

    The reference records a running-max snapshot after every visit; the one consumer on the
    forward path, stabilization_positions (src/analysis.py:39-78), needs only the block after
    which each row's max held its final value, which the kernel records directly
    (`positions`, 1-based key blocks, shape [..., Nq]) together with each query block's local
    key block -- so the analysis runs at any context length.
    """

    q_block: int
    positions: torch.Tensor
    local_blocks: list
    # the reference's per-visit records when the run kept them (state_trace): snapshots
    # [..., Nq, T_c] (running max after each visit position, NaN past the visible blocks) and the
    # visit order of every query block (1-based key blocks, the device scheduler's order)
    snapshots: torch.Tensor | None = None
    orders: list | None = None

    @classmethod
    def from_run(cls, p: "AttentionProblem", stab, snapshots=None, variant="vfa", reorder=True,
                 n_sink=1, n_local=1) -> "DeviceTrace":
        b = p.blocks
        local = [min((i * b.q_block - 1) // b.k_block + 1, b.t_c) for i in range(1, b.t_r + 1)]
        orders = None
        if snapshots is not None:
            orders = [tile_schedule(i, b.q_block, b.k_block, b.t_c, p.causal, n_sink, n_local, reorder,
                                    variant)[0] for i in range(1, b.t_r + 1)]
        return cls(q_block=b.q_block, positions=stab, local_blocks=local, snapshots=snapshots, orders=orders)

    @property
    def records(self) -> list:
        """Per query block, [(pos, block, m after the visit)] like the reference's
        StateTrace.records (src/core.py:35-54); needs the snapshots."""
        if self.snapshots is None:
            raise ValueError("this trace has no per-visit snapshots (run with state_trace=True)")
        snap = self.snapshots.reshape(-1, self.snapshots.shape[-2], self.snapshots.shape[-1])
        snap = snap.double().cpu().numpy()
        out = []
        for bi, order in enumerate(self.orders):
            rows = snap[:, bi * self.q_block:(bi + 1) * self.q_block]
            out.append([(pos, j, rows[..., pos].reshape(-1)) for pos, j in enumerate(order)])
        return out


@dataclass
class StabilizationReport:
    """src/analysis.py:30-37."""

    positions: np.ndarray
    frac_sink: float
    frac_local: float
    frac_other: float

    def frac_sink_or_local(self) -> float:
        return self.frac_sink + self.frac_local


def stabilization_positions(trace: DeviceTrace, final_m=None) -> StabilizationReport:
    """Fractions of rows whose running max stabilised in the sink block, the local block or
    elsewhere (src/analysis.py:39-78), from a DeviceTrace of one or more heads.

    final_m: as in the reference, check the trace against maxima obtained elsewhere: the
    position of a row is the block of its first visit whose running-max snapshot equals
    final_m exactly (ValueError if none does); needs a trace with snapshots. Without final_m
    the kernel's own positions are used (= the snapshots against their last value)."""
    qb = trace.q_block
    if final_m is None:
        pos = trace.positions.to(torch.int64).cpu().numpy()
    else:
        if trace.snapshots is None:
            raise ValueError("final_m needs a trace with per-visit snapshots (state_trace=True)")
        snap = trace.snapshots.double().cpu().numpy()
        fm = np.asarray(final_m.cpu() if isinstance(final_m, torch.Tensor) else final_m, dtype=np.float64)
        fm = np.broadcast_to(fm.reshape(*fm.shape), snap.shape[:-1])
        pos = np.zeros(snap.shape[:-1], dtype=np.int64)
        settled = np.zeros(snap.shape[:-1], dtype=bool)
        for bi, order in enumerate(trace.orders):
            rs = slice(bi * qb, (bi + 1) * qb)
            pos[..., rs] = order[-1]
            for p_i, j in enumerate(order):
                hit = ~settled[..., rs] & (snap[..., rs, p_i] == fm[..., rs])
                pos[..., rs][hit] = j
                settled[..., rs] |= hit
        if not settled.all():
            raise ValueError("running max never reached its final value")
    nq = pos.shape[-1]
    local = np.repeat(np.asarray(trace.local_blocks, dtype=np.int64), qb)[:nq]
    sink = pos == 1
    loc = (pos == local) & (local != 1)
    n = pos.size
    return StabilizationReport(positions=pos, frac_sink=float(sink.sum()) / n,
                               frac_local=float(loc.sum()) / n,
                               frac_other=float((~sink & (pos != local)).sum()) / n)


# the reference-shaped fa_forward / vfa_forward keep the per-visit StateTrace snapshots (one
# float per row and key block) up to this many entries, i.e. for the reference's desk-scale
# problems; larger problems return the per-row stabilization positions only
SNAPSHOT_LIMIT = 1 << 24


def _keep_snapshots(p: AttentionProblem) -> bool:
    heads = 1 if p.q.dim() == 2 else p.q.shape[0] * p.q.shape[1]
    return heads * p.blocks.seq_len_q * p.blocks.t_c <= SNAPSHOT_LIMIT


def _counters(st, p: AttentionProblem, variant: str) -> OpCounters:
    return OpCounters.from_stats(variant, st, p.blocks.q_block, p.blocks.k_block, p.blocks.head_dim)


def _monitor(st, monitor: bool) -> OverflowMonitor:
    """OverflowMonitor from the device counters (src/vfa.py:109-135). The reference records
    the argument statistics on every call and the calibration gap only with monitor=True;
    the device records all of them only with monitor=True (the counting costs kernel time),
    so without it exp_arg_max is -inf and the counts are 0."""
    m = OverflowMonitor()
    if monitor:
        m.count_over_f16 = st["count_over_f16"]
        m.count_over_f32 = st["count_over_f32"]
        m.exp_arg_max = st["exp_arg_max"]
        m.calibration_gap = st["calibration_gap"]
    return m


def fa_forward(p: AttentionProblem, order_hook=None):
    """Baseline online softmax, rescale on every block (src/fa.py:28-61).

    Returns (O, counters, DeviceTrace) with `.lse`. order_hook (a test-only
    permutation hook in the reference) is not supported on the GPU path.
    """
    if order_hook is not None:
        raise ValueError("order_hook is not supported by the GPU fa_forward")
    out, lse, st = _run(p, "fa", stab_trace=True, state_trace=_keep_snapshots(p))
    trace = DeviceTrace.from_run(p, st["stab_block"], st.get("m_trace"), "fa", False)
    return ForwardResult((out, _counters(st, p, "fa"), trace), lse, st)


def vfa_forward(p: AttentionProblem, kind: str = "sabsmax", reorder: bool = True,
                use_m_init: bool = True, qkind: str = "row_wise", tc1: int | None = None,
                monitor: bool = False, *, n_sink: int = 1, n_local: int = 1):
    """Frozen-max pass with m-initialisation (src/vfa.py:156-223).

    Returns (O, counters, DeviceTrace, overflow_monitor) with `.lse`.
    """
    if kind not in _lib.KEY_REPRS:
        raise ValueError(f"unknown key representation {kind!r}")
    if qkind not in _lib.QUERY_REPRS:
        raise ValueError(f"unknown query representation {qkind!r}")
    if tc1 is not None and not (1 <= tc1 <= p.t_c):
        raise ValueError(f"tc1 must be in 1..{p.t_c}, got {tc1}")
    snaps = _keep_snapshots(p)
    out, lse, st = _run(p, "vfa", kind=kind, reorder=reorder, use_m_init=use_m_init, qkind=qkind,
                        tc1=tc1, n_sink=n_sink, n_local=n_local, monitor=monitor, stab_trace=True,
                        state_trace=snaps)
    trace = DeviceTrace.from_run(p, st["stab_block"], st.get("m_trace"), "vfa", reorder, n_sink, n_local)
    return ForwardResult((out, _counters(st, p, "vfa"), trace, _monitor(st, monitor)), lse, st)


def vsa_forward(p: AttentionProblem, cfg: SkipConfig, kind: str = "sabsmax", qkind: str = "row_wise",
                tc1: int | None = None, monitor: bool = False, *, n_sink: int = 1, n_local: int = 1):
    """Frozen max + BLASST block skipping (src/sparse.py:256-329).

    Returns (O, counters, SkipStats, overflow_monitor) with `.lse`.
    """
    if cfg.granularity != "block":
        raise ValueError("vsa_forward requires block granularity")
    if kind not in _lib.KEY_REPRS:
        raise ValueError(f"unknown key representation {kind!r}")
    if tc1 is not None and not (1 <= tc1 <= p.t_c):
        raise ValueError(f"tc1 must be in 1..{p.t_c}, got {tc1}")
    out, lse, st = _run(p, "vsa", kind=kind, qkind=qkind, tc1=tc1, n_sink=n_sink, n_local=n_local,
                        lam=cfg.lam, monitor=monitor)
    stats = SkipStats(blocks_visited=st["visited"], blocks_skipped=st["skipped"],
                      blocks_processed=st["special"] + st["frozen"],
                      processed_special=st["special"], processed_frozen=st["frozen"])
    return ForwardResult((out, _counters(st, p, "vsa"), stats, _monitor(st, monitor)), lse, st)


def _skip_stats(st, qb, row_slots=False) -> SkipStats:
    return SkipStats(blocks_visited=st["visited"], blocks_skipped=st["skipped"],
                     rows_masked=st["rows_masked"], row_slots=st["visited"] * qb if row_slots else 0,
                     rescales_elided=st["elided"], blocks_processed=st["special"] + st["frozen"])


def blasst_forward(p: AttentionProblem, cfg: SkipConfig, order: str = "sequential"):
    """Threshold block skipping on the baseline recurrence (src/sparse.py:112-152).

    order='sink_local' visits the sink and local blocks first (the VFA order) with the
    skip rule unchanged. Returns (O, counters, SkipStats) with `.lse`.
    """
    if cfg.granularity != "block":
        raise ValueError("blasst_forward requires block granularity")
    if order not in ("sequential", "sink_local"):
        raise ValueError(f"unknown order {order!r}")
    out, lse, st = _run(p, "blasst", lam=cfg.lam, reorder=order == "sink_local")
    b = p.blocks
    c = OpCounters.from_stats("blasst", st, b.q_block, b.k_block, b.head_dim)
    return ForwardResult((out, c, _skip_stats(st, b.q_block)), lse, st)


def blasst_fa4_forward(p: AttentionProblem, cfg: SkipConfig):
    """Block skipping plus rescale elision when no row max rises by more than tau*ln2
    (src/sparse.py:155-203). Returns (O, counters, SkipStats) with `.lse`."""
    if cfg.granularity != "block":
        raise ValueError("blasst_fa4_forward requires block granularity")
    out, lse, st = _run(p, "blasst_fa4", lam=cfg.lam, tau=cfg.tau)
    b = p.blocks
    c = OpCounters.from_stats("blasst_fa4", st, b.q_block, b.k_block, b.head_dim)
    return ForwardResult((out, c, _skip_stats(st, b.q_block)), lse, st)


def blasst_rowskip_forward(p: AttentionProblem, cfg: SkipConfig):
    """Row-granular thresholding: suppressed rows contribute zero mass
    (src/sparse.py:206-253). Returns (O, counters, SkipStats) with `.lse`."""
    if cfg.granularity != "row":
        raise ValueError("blasst_rowskip_forward requires row granularity")
    out, lse, st = _run(p, "blasst_rowskip", lam=cfg.lam)
    b = p.blocks
    c = OpCounters.from_stats("blasst_rowskip", st, b.q_block, b.k_block, b.head_dim)
    return ForwardResult((out, c, _skip_stats(st, b.q_block, row_slots=True)), lse, st)


def precompute_kreprs(p: AttentionProblem, kind: str, tc1: int | None = None, *, out=None,
                      first_block: int = 0) -> torch.Tensor:
    """Key-block representations on the GPU (src/vfa.py:79-88): bf16 [..., n_blocks, d].

    Incremental use for an append-only K cache: pass the previous result as
    `out` and the 0-based first block whose keys changed as `first_block`; only blocks from
    there on are recomputed (vfa_krepr_range).
    """
    if kind not in _lib.KEY_REPRS:
        raise ValueError(f"unknown key representation {kind!r}")
    tc1 = p.t_c if tc1 is None else tc1
    if not (1 <= tc1 <= p.t_c):
        raise ValueError(f"tc1 must be in 1..{p.t_c}, got {tc1}")
    k = p.k if p.k.dim() == 4 else p.k.view(1, 1, *p.k.shape)
    q = p.q if p.q.dim() == 4 else p.q.view(1, 1, *p.q.shape)
    prm = _params(q, k, k, q, variant="vfa", causal=p.causal, q_block=p.blocks.q_block,
                  k_block=p.blocks.k_block, scale=p.scale, kind=kind, qkind="row_wise", reorder=True,
                  use_m_init=True, tc1=tc1, n_sink=1, n_local=1, lam=None, monitor=False)
    shape = (k.shape[0], k.shape[1], tc1, k.shape[3])
    if out is None:
        if first_block:
            raise ValueError("first_block > 0 needs the previous representations as `out`")
        out = torch.empty(shape, dtype=torch.bfloat16, device=k.device)
    else:
        out = out if out.dim() == 4 else out.view(1, 1, *out.shape)
        if tuple(out.shape) != shape or out.dtype != torch.bfloat16 or not out.is_contiguous():
            raise ValueError(f"out must be a contiguous bf16 tensor of shape {shape}")
    lib = _lib.load()
    with torch.cuda.device(k.device):
        rc = lib.vfa_krepr_range(ctypes.byref(prm), k.data_ptr(), out.data_ptr(), int(first_block),
                                 ctypes.c_void_p(torch.cuda.current_stream(k.device).cuda_stream))
    if rc:
        _raise_for(rc)
    return out if p.k.dim() == 4 else out[0, 0]


def tile_schedule(i, q_block, k_block, t_c, causal, n_sink=1, n_local=1, reorder=True, variant="vfa"):
    """The device tile scheduler's visit order and exact-update set for query block i."""
    return _lib.schedule(i, q_block, k_block, t_c, causal, n_sink, n_local, reorder, variant)
