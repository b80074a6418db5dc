"""Multi-GPU partitioning of the attention forward by KV-head group.

Units are independent (query blocks and heads never interact), so rank r of
`world` owns a contiguous block of KV heads and their GQA query heads: K/V are never
replicated and no collective runs in the steady state. `gather_heads` concatenates the
per-rank O / LSE shards along the head axis (NCCL all_gather on GPUs; gloo in the CPU
tests) for verification only.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class HeadShard:
    kv0: int
    kv1: int  # exclusive
    q0: int
    q1: int  # exclusive


def kv_head_shard(rank: int, world: int, heads_q: int, heads_kv: int) -> HeadShard:
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    if heads_q % heads_kv:
        raise ValueError("heads_q must be a multiple of heads_kv")
    if heads_kv % world:
        raise ValueError(f"world size {world} must divide heads_kv={heads_kv}")
    per = heads_kv // world
    grp = heads_q // heads_kv
    kv0 = rank * per
    return HeadShard(kv0, kv0 + per, kv0 * grp, (kv0 + per) * grp)


def shard_inputs(q, k, v, shard: HeadShard):
    """Slice [B, H, L, d] tensors to a rank's heads (contiguous copies)."""
    return (q[:, shard.q0:shard.q1].contiguous(), k[:, shard.kv0:shard.kv1].contiguous(),
            v[:, shard.kv0:shard.kv1].contiguous())


def gather_heads(x, world: int):
    """all_gather a per-rank [B, h, ...] shard and concatenate along dim 1."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return x
    if dist.get_backend() == "gloo" and x.is_cuda:  # gloo gathers host tensors
        parts = [torch.empty_like(x, device="cpu") for _ in range(world)]
        dist.all_gather(parts, x.contiguous().cpu())
        return torch.cat(parts, 1).to(x.device)
    parts = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(parts, x.contiguous())
    return torch.cat(parts, 1)
