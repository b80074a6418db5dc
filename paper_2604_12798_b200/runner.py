"""GPU backend for the reference's `run` / `compare` commands on VFT1 dumps (SURVEY.md §8f
rank 4; src/cli.py:213-319, 383-445): real-model Q/K/V written as `q.vft`, `k.vft`, `v.vft`
(src/cli.py:213-221) run through the B200 kernels, and the result is reported in the
reference's JSON schema {meta, values, counters, stats, monitor} plus device timing.

Inputs are rounded to bf16 (the kernels' input precision; the report says so). Errors map to
the reference CLI's exit codes (src/cli.py:69-72): ConfigError 2, DataError / VFT1 errors 3,
numerical (FullyMaskedRowError, NormalizerUnderflowError) 4.
"""

from __future__ import annotations

import hashlib
import json
import time
from pathlib import Path

import numpy as np
import torch

from . import api, vft1

EXIT_OK, EXIT_CONFIG, EXIT_DATA, EXIT_NUMERICAL = 0, 2, 3, 4
VARIANTS = ("fa", "vfa", "blasst", "blasst_swa", "blasst_fa4", "blasst_rowskip", "vsa")  # src/cli.py:60-67
# the reference's run defaults (src/cli.py:83-105)
DEFAULTS = {"q_block": 64, "k_block": 64, "causal": False, "variant": "fa", "repr": "sabsmax",
            "q_repr": "row_wise", "lambda": None, "tau": 0.0, "reorder": True, "m_init": True,
            "monitor": False, "tc1": None}


class ConfigError(ValueError):
    pass


class DataError(ValueError):
    pass


def load_tensors(data_dir):
    """q.vft / k.vft / v.vft of a dump directory as float64 matrices (src/cli.py:213-221)."""
    d = Path(data_dir)
    out = []
    for name in ("q", "k", "v"):
        path = d / f"{name}.vft"
        if not path.exists():
            raise DataError(f"missing tensor file {path}")
        out.append(vft1.read_matrix(path))
    return tuple(out)


def problem_from(cfg: dict, q, k, v) -> api.AttentionProblem:
    """src/cli.py:224-240: shape checks and the block geometry, as DataError."""
    if k.shape[1] != q.shape[1] or v.shape[1] != q.shape[1] or k.shape[0] != v.shape[0]:
        raise DataError(f"inconsistent tensor shapes: q{q.shape} k{k.shape} v{v.shape}")
    try:
        blocks = api.BlockSpec(q.shape[0], k.shape[0], q.shape[1], cfg["q_block"], cfg["k_block"])
        return api.AttentionProblem(torch.from_numpy(q), torch.from_numpy(k), torch.from_numpy(v),
                                    blocks=blocks, causal=cfg["causal"])
    except ValueError as e:
        raise DataError(str(e)) from e


def execute(cfg: dict, p: api.AttentionProblem):
    """The variant switch of src/cli.py:243-286 on the GPU path: (out, counters, stats, monitor)."""
    v = cfg["variant"]
    if v == "fa":
        out, counters, _ = api.fa_forward(p)
        return out, counters, None, None
    if v == "vfa":
        out, counters, _, mon = api.vfa_forward(p, kind=cfg["repr"], reorder=cfg["reorder"],
                                                use_m_init=cfg["m_init"], qkind=cfg["q_repr"],
                                                tc1=cfg["tc1"], monitor=cfg["monitor"])
        return out, counters, None, mon
    if v in ("blasst", "blasst_swa"):
        out, counters, stats = api.blasst_forward(p, api.SkipConfig(lam=cfg["lambda"]),
                                                  order="sink_local" if v == "blasst_swa" else "sequential")
        return out, counters, stats, None
    if v == "blasst_fa4":
        out, counters, stats = api.blasst_fa4_forward(p, api.SkipConfig(lam=cfg["lambda"], tau=float(cfg["tau"])))
        return out, counters, stats, None
    if v == "blasst_rowskip":
        out, counters, stats = api.blasst_rowskip_forward(p, api.SkipConfig(lam=cfg["lambda"], granularity="row"))
        return out, counters, stats, None
    if v == "vsa":
        out, counters, stats, mon = api.vsa_forward(p, api.SkipConfig(lam=cfg["lambda"]), kind=cfg["repr"],
                                                    qkind=cfg["q_repr"], tc1=cfg["tc1"], monitor=cfg["monitor"])
        return out, counters, stats, mon
    raise ConfigError(f"variant: unknown {v!r} (GPU variants: {', '.join(VARIANTS)})")


def checksum(m: np.ndarray) -> str:
    """src/cli.py:206-210 (shape + float64 bytes)."""
    h = hashlib.sha256()
    h.update(str(m.shape).encode())
    h.update(np.ascontiguousarray(m, dtype=np.float64).tobytes())
    return h.hexdigest()


def rel_err(a: np.ndarray, b: np.ndarray):
    """src/cli.py:322-327: row-wise ||a - b||_inf / ||b||_inf, (max, mean)."""
    diff = np.abs(a - b).max(axis=1)
    rel = diff / np.maximum(np.abs(b).max(axis=1), np.finfo(np.float64).tiny)
    return float(rel.max()), float(rel.mean())


def _config(**kw) -> dict:
    cfg = dict(DEFAULTS)
    for key, val in kw.items():
        key = "lambda" if key == "lam" else key
        if key not in cfg:
            raise ConfigError(f"unknown option {key!r}")
        cfg[key] = val
    if cfg["variant"] not in VARIANTS:
        raise ConfigError(f"variant: unknown {cfg['variant']!r} (GPU variants: {', '.join(VARIANTS)})")
    if cfg["lambda"] is not None and not (0.0 < cfg["lambda"] <= 1.0):
        raise ConfigError(f"lambda must be in (0, 1] or None, got {cfg['lambda']}")
    return cfg


def _timed(cfg, p):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = execute(cfg, p)
    e1.record()
    torch.cuda.synchronize()
    return res, e0.elapsed_time(e1)


def _flops(p: api.AttentionProblem) -> float:
    lq, lk, d = p.blocks.seq_len_q, p.blocks.seq_len_k, p.blocks.head_dim
    pairs = lq * (lq + 1) / 2 if p.causal else lq * lk
    return 4.0 * pairs * d


def _report(command, cfg, values, counters=None, stats=None, monitor=None, wall=0.0):
    return {
        "meta": {"command": command, "config": dict(sorted(cfg.items())), "backend": "b200",
                 "input_precision": "bf16", "timestamp": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
                 "wall_time_s": wall},
        "values": values,
        "counters": counters.as_dict() if counters is not None else None,
        "stats": stats.as_dict() if stats is not None else None,
        "monitor": None if monitor is None else {"exp_arg_max": monitor.exp_arg_max,
                                                 "count_over_f16": monitor.count_over_f16,
                                                 "count_over_f32": monitor.count_over_f32,
                                                 "calibration_gap": monitor.calibration_gap},
    }


def _write(report, path):
    if path is None:
        return
    text = json.dumps(report, indent=2, sort_keys=True)
    if path == "-":
        print(text)
    else:
        Path(path).write_text(text + "\n")


def run(data_dir, *, report=None, out=None, **kw) -> dict:
    """The reference's `run` (src/cli.py:383-407) on the GPU: returns the report dict and
    optionally writes it (JSON) and the output (VFT1 float64) to disk."""
    cfg = _config(**kw)
    q, k, v = load_tensors(data_dir)
    p = problem_from(cfg, q, k, v)
    t0 = time.perf_counter()
    (o, counters, stats, mon), ms = _timed(cfg, p)
    o64 = o.double().cpu().numpy()
    wall = time.perf_counter() - t0
    values = {"variant": cfg["variant"], "output_checksum": checksum(o64), "output_shape": list(o64.shape),
              "device_ms": ms, "tflops": _flops(p) / (ms * 1e-3) / 1e12}
    if stats is not None:
        values.update(block_sparsity=stats.block_sparsity, row_sparsity=stats.row_sparsity,
                      rescale_skip_rate=stats.rescale_skip_rate)
    rep = _report("run", cfg, values, counters, stats, mon, wall)
    _write(rep, report)
    if out is not None:
        vft1.write_matrix(out, o64)
    return rep


def compare(data_dir, variant_b, *, lambda_b=None, tau_b=None, report=None, **kw) -> dict:
    """The reference's `compare` (src/cli.py:410-445) on the GPU: two variants on one dump."""
    cfg_a = _config(**kw)
    cfg_b = dict(cfg_a, variant=variant_b)
    if lambda_b is not None:
        cfg_b["lambda"] = lambda_b
    if tau_b is not None:
        cfg_b["tau"] = tau_b
    cfg_b = _config(**cfg_b)
    q, k, v = load_tensors(data_dir)
    p = problem_from(cfg_a, q, k, v)
    t0 = time.perf_counter()
    (oa, ca, sa, _), _ = _timed(cfg_a, p)
    (ob, cb, sb, _), _ = _timed(cfg_b, p)
    wall = time.perf_counter() - t0
    a64, b64 = oa.double().cpu().numpy(), ob.double().cpu().numpy()
    max_rel, mean_rel = rel_err(a64, b64)
    da, db = ca.as_dict(), cb.as_dict()
    values = {"variant_a": cfg_a["variant"], "variant_b": cfg_b["variant"], "checksum_a": checksum(a64),
              "checksum_b": checksum(b64), "max_rel_diff": max_rel, "mean_rel_diff": mean_rel,
              "counter_delta": {key: db[key] - da[key] for key in da},
              "sparsity_a": sa.block_sparsity if sa else None, "sparsity_b": sb.block_sparsity if sb else None}
    cfg_dump = dict(cfg_a, variant_b=cfg_b["variant"])
    rep = _report("compare", cfg_dump, values, wall=wall)
    _write(rep, report)
    return rep


def exit_code(exc: BaseException) -> int:
    """Map an exception to the reference CLI's exit codes (src/cli.py:636-644)."""
    if isinstance(exc, ConfigError):
        return EXIT_CONFIG
    if isinstance(exc, (DataError, vft1.TensorIOError)):
        return EXIT_DATA
    if isinstance(exc, (api.FullyMaskedRowError, api.NormalizerUnderflowError)):
        return EXIT_NUMERICAL
    if isinstance(exc, ValueError):
        return EXIT_CONFIG
    raise exc
