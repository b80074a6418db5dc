"""B200-native (sm_100a) VFA / VSA attention forward — drop-in for the reference's
`vfa_lab` attention entry points (arXiv 2604.12798).

Compute runs in libvfa_b200.so (hand-written tcgen05/TMEM/TMA kernels, C ABI in
include/vfa_b200.h). This package is the host-side mirror of the reference API.
"""

from ._lib import KEY_REPRS, QUERY_REPRS, LibraryNotBuilt
from .api import (AttentionProblem, BlockSpec, DeviceTrace, ForwardResult, FullyMaskedRowError,
                  KernelError, NormalizerUnderflowError, OpCounters, OverflowMonitor, SkipConfig,
                  SkipStats, StabilizationReport, attention_forward, attention_forward_host,
                  blasst_fa4_forward, blasst_forward, blasst_rowskip_forward, check_status,
                  fa_forward, precompute_kreprs, stabilization_positions, stats_dict, tile_schedule,
                  vfa_forward, vsa_forward)

__version__ = "0.1.0"

__all__ = [
    "AttentionProblem", "BlockSpec", "DeviceTrace", "ForwardResult", "FullyMaskedRowError",
    "KEY_REPRS", "KernelError", "LibraryNotBuilt", "NormalizerUnderflowError", "OpCounters",
    "OverflowMonitor", "QUERY_REPRS", "SkipConfig", "SkipStats", "StabilizationReport",
    "attention_forward", "attention_forward_host", "blasst_fa4_forward", "blasst_forward",
    "blasst_rowskip_forward", "check_status", "fa_forward", "precompute_kreprs",
    "stabilization_positions", "stats_dict", "tile_schedule", "vfa_forward", "vsa_forward",
]
