"""Multi-GPU partitioning of the attention forward by (batch, KV head) units.

Units are independent (query blocks and heads never interact). A unit is one
batch entry's KV head together with its GQA query heads; the B * Hkv units are numbered
batch-major (u = b * Hkv + kvh) and rank r of `world` owns the contiguous range [u0, u1)
(as even as possible: the first B*Hkv % world ranks take one unit more). K/V are never
replicated and no collective runs in the steady state.

A rank's range is a list of rectangular pieces (one per batch entry it touches), each a
strided view of the caller's [B, H, L, d] tensors that the kernel consumes directly (no
copies). `gather_units` collects the per-rank unit-major O / LSE buffers for verification
only (NCCL all_gather on GPUs; gloo in the CPU tests), padding ranks with fewer units.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class UnitShard:
    u0: int
    u1: int  # exclusive
    batch: int
    heads_kv: int
    group: int  # query heads per KV head

    @property
    def units(self) -> int:
        return self.u1 - self.u0

    @property
    def pieces(self) -> list:
        """[(b, kv0, kv1)] rectangular pieces of the range, in unit order."""
        out = []
        for b in range(self.u0 // self.heads_kv, (self.u1 + self.heads_kv - 1) // self.heads_kv):
            kv0 = max(self.u0 - b * self.heads_kv, 0)
            kv1 = min(self.u1 - b * self.heads_kv, self.heads_kv)
            if kv1 > kv0:
                out.append((b, kv0, kv1))
        return out


def unit_shard(rank: int, world: int, batch: int, heads_q: int, heads_kv: int) -> UnitShard:
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    if heads_q % heads_kv:
        raise ValueError("heads_q must be a multiple of heads_kv")
    total = batch * heads_kv
    if world > total:
        raise ValueError(f"world size {world} exceeds the {total} (batch, KV head) units")
    base, extra = divmod(total, world)
    u0 = rank * base + min(rank, extra)
    u1 = u0 + base + (1 if rank < extra else 0)
    return UnitShard(u0, u1, batch, heads_kv, heads_q // heads_kv)


def kv_head_shard(rank: int, world: int, heads_q: int, heads_kv: int) -> UnitShard:
    """Batch-1 special case (the C2 / C4 configs): a contiguous block of KV heads."""
    return unit_shard(rank, world, 1, heads_q, heads_kv)


def shard_views(q, k, v, shard: UnitShard) -> list:
    """Per piece: (q, k, v) strided views [1, n*group, L, d] / [1, n, L, d] of the caller's
    [B, H, L, d] tensors (the kernel takes any strides with a contiguous head dimension)."""
    g = shard.group
    return [(q[b:b + 1, kv0 * g:kv1 * g], k[b:b + 1, kv0:kv1], v[b:b + 1, kv0:kv1])
            for b, kv0, kv1 in shard.pieces]


def shard_inputs(q, k, v, shard: UnitShard):
    """The rank's units as contiguous tensors when the range is one piece (batch-1 configs)."""
    pieces = shard_views(q, k, v, shard)
    if len(pieces) != 1:
        raise ValueError("the unit range spans several batch entries: use shard_views")
    return tuple(x.contiguous() for x in pieces[0])


def unit_major(x, heads_kv: int):
    """View a [B, H, ...] tensor as [B * Hkv, H / Hkv, ...] (unit-major; contiguous input)."""
    return x.reshape(x.shape[0] * heads_kv, x.shape[1] // heads_kv, *x.shape[2:])


def gather_units(x_units, shard: UnitShard, world: int):
    """all_gather every rank's unit-major [units, ...] buffer (padded to the largest range)
    and return all B * Hkv units in order."""
    import torch
    import torch.distributed as dist
    total = shard.batch * shard.heads_kv
    if world == 1:
        return x_units
    base, extra = divmod(total, world)
    width = base + (1 if extra else 0)
    pad = torch.zeros((width, *x_units.shape[1:]), dtype=x_units.dtype, device=x_units.device)
    pad[: x_units.shape[0]] = x_units
    host = dist.get_backend() == "gloo" and pad.is_cuda  # gloo gathers host tensors
    src = pad.cpu() if host else pad
    parts = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(parts, src)
    counts = [base + (1 if r < extra else 0) for r in range(world)]
    out = torch.cat([p[:n] for p, n in zip(parts, counts)], 0)
    return out.to(x_units.device) if host else out


def gather_heads(x, world: int):
    """Batch-1, evenly divisible case: all_gather [1, h, ...] shards along the head axis."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return x
    if dist.get_backend() == "gloo" and x.is_cuda:
        parts = [torch.empty_like(x, device="cpu") for _ in range(world)]
        dist.all_gather(parts, x.contiguous().cpu())
        return torch.cat(parts, 1).to(x.device)
    parts = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(parts, x.contiguous())
    return torch.cat(parts, 1)
