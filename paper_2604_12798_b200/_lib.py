"""ctypes binding of the C ABI declared in include/vfa_b200.h (libvfa_b200.so).

The library is built in-tree (paper_2604_12798_b200/libvfa_b200.so) by
`paper_2604_12798_b200.build.build()`. There is no fallback: if the library is
missing, every GPU entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

LIB_NAME = "libvfa_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)
# experiments only (e.g. tuning-knob sweeps): load an alternative in-tree build
LIB_PATH = os.environ.get("VFA_B200_LIB", LIB_PATH)

VFA_OK = 0
VFA_ERR_CONFIG = 2
VFA_ERR_DATA = 3
VFA_ERR_NUMERICAL = 4
VFA_ERR_CUDA = 5

VARIANTS = {"fa": 0, "vfa": 1, "vsa": 2, "blasst": 3, "blasst_fa4": 4, "blasst_rowskip": 5}
KEY_REPRS = ("sabsmax", "k_max", "k_mean", "k_absmax_unsigned")  # src/vfa.py:39
QUERY_REPRS = ("row_wise", "q_absmax", "q_sabsmax", "q_mean")  # src/vfa.py:40

(STAT_VISITED, STAT_SKIPPED, STAT_SPECIAL, STAT_FROZEN, STAT_OVER_F32, STAT_OVER_F16, STAT_ELIDED,
 STAT_ROWS_MASKED, STAT_EXP_ARG_MAX, STAT_GAP_NEG_MIN, STAT_GAP_MAX, STAT_GAP_SUM, STAT_GAP_BELOW,
 STAT_GAP_ROWS) = range(14)
STAT_COUNT = 14
STATUS_FLAGS, STATUS_UNDERFLOW_ROW, STATUS_MASKED_ROW, STATUS_NONFINITE_ROWS = range(4)
STATUS_COUNT = 4

# every symbol include/vfa_b200.h declares
EXPORTS = ("vfa_check_params", "vfa_workspace_bytes", "vfa_fwd", "vfa_krepr", "vfa_schedule",
           "vfa_status_code", "vfa_last_error", "vfa_version", "vfa_debug_trace",
           "vfa_host_scratch_bytes", "vfa_fwd_host", "vfa_krepr_range", "vfa_fwd_rebased",
           "vfa_fwd_state_trace")


class VfaParams(ctypes.Structure):
    """Mirror of `VfaParams` in include/vfa_b200.h (field order and types must match)."""

    _fields_ = [
        ("batch", ctypes.c_int64), ("heads_q", ctypes.c_int64), ("heads_kv", ctypes.c_int64),
        ("seq_q", ctypes.c_int64), ("seq_k", ctypes.c_int64), ("head_dim", ctypes.c_int64),
        ("q_stride", ctypes.c_int64 * 3), ("k_stride", ctypes.c_int64 * 3),
        ("v_stride", ctypes.c_int64 * 3), ("o_stride", ctypes.c_int64 * 3),
        ("scale", ctypes.c_double),
        ("causal", ctypes.c_int32), ("q_block", ctypes.c_int32), ("k_block", ctypes.c_int32),
        ("variant", ctypes.c_int32), ("kind", ctypes.c_int32), ("qkind", ctypes.c_int32),
        ("reorder", ctypes.c_int32), ("use_m_init", ctypes.c_int32), ("tc1", ctypes.c_int32),
        ("n_sink", ctypes.c_int32), ("n_local", ctypes.c_int32), ("monitor", ctypes.c_int32),
        ("lam", ctypes.c_double),
        ("krepr_precomputed", ctypes.c_int32), ("softmax_split", ctypes.c_int32),
        ("tau", ctypes.c_double),
        ("cta_pair", ctypes.c_int32), ("reserved", ctypes.c_int32),
    ]


_lib = None
_lock = threading.Lock()


class LibraryNotBuilt(RuntimeError):
    pass


def bind(path: str):
    """ctypes.CDLL of a libvfa_b200 build at `path` with every C-ABI signature set."""
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER(VfaParams)
    vp = ctypes.c_void_p
    lib.vfa_check_params.argtypes = [P]
    lib.vfa_check_params.restype = ctypes.c_int
    lib.vfa_workspace_bytes.argtypes = [P]
    lib.vfa_workspace_bytes.restype = ctypes.c_size_t
    lib.vfa_fwd.argtypes = [P, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp, vp, vp, vp, vp]
    lib.vfa_fwd.restype = ctypes.c_int
    lib.vfa_fwd_rebased.argtypes = [P, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp, vp, vp, vp]
    lib.vfa_fwd_rebased.restype = ctypes.c_int
    lib.vfa_fwd_state_trace.argtypes = [P, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp, vp, vp, vp, vp]
    lib.vfa_fwd_state_trace.restype = ctypes.c_int
    lib.vfa_host_scratch_bytes.argtypes = [P, ctypes.c_int, ctypes.c_int]
    lib.vfa_host_scratch_bytes.restype = ctypes.c_size_t
    lib.vfa_fwd_host.argtypes = [P, vp, vp, vp, vp, vp, vp, ctypes.c_size_t, vp, vp, ctypes.c_int, ctypes.c_int,
                                 vp]
    lib.vfa_fwd_host.restype = ctypes.c_int
    lib.vfa_krepr.argtypes = [P, vp, vp, vp]
    lib.vfa_krepr_range.argtypes = [P, vp, vp, ctypes.c_int, vp]
    lib.vfa_krepr_range.restype = ctypes.c_int
    lib.vfa_krepr.restype = ctypes.c_int
    lib.vfa_schedule.argtypes = [ctypes.c_int] * 9 + [ctypes.POINTER(ctypes.c_int),
                                                     ctypes.POINTER(ctypes.c_ubyte), ctypes.c_int]
    lib.vfa_schedule.restype = ctypes.c_int
    lib.vfa_status_code.argtypes = [ctypes.POINTER(ctypes.c_uint)]
    lib.vfa_status_code.restype = ctypes.c_int
    lib.vfa_last_error.argtypes = []
    lib.vfa_last_error.restype = ctypes.c_char_p
    lib.vfa_debug_trace.argtypes = [vp]
    lib.vfa_debug_trace.restype = ctypes.c_int
    lib.vfa_version.argtypes = []
    lib.vfa_version.restype = ctypes.c_char_p
    return lib


def load():
    """Load libvfa_b200.so (raises LibraryNotBuilt if absent — there is no CPU fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LibraryNotBuilt(
                f"{LIB_PATH} not found: run `python -c 'import __graft_entry__ as g; g.build()'`")
        _lib = bind(LIB_PATH)
        return _lib


def key_to_float(key: int) -> float:
    """Decode an order-preserving float key of the stats word (include/vfa_b200.h); NaN if unset."""
    import struct
    key &= 0xFFFFFFFF
    if key == 0:
        return float("nan")
    bits = key ^ 0x80000000 if key & 0x80000000 else (~key) & 0xFFFFFFFF
    return struct.unpack("<f", struct.pack("<I", bits))[0]


def last_error() -> str:
    return load().vfa_last_error().decode()


def schedule(i, q_block, k_block, t_c, causal, n_sink=1, n_local=1, reorder=True, variant="vfa"):
    """Host mirror of the device tile scheduler: returns (order tuple, special frozenset)."""
    lib = load()
    cap = max(t_c, 1)
    order = (ctypes.c_int * cap)()
    spec = (ctypes.c_ubyte * cap)()
    n = lib.vfa_schedule(i, q_block, k_block, t_c, int(bool(causal)), n_sink, n_local,
                         int(bool(reorder)), VARIANTS[variant], order, spec, cap)
    if n < 0:
        raise ValueError(last_error())
    blocks = tuple(order[p] for p in range(n))
    return blocks, frozenset(order[p] for p in range(n) if spec[p])
