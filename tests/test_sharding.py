"""Multi-process (gloo, world size 2) test of the (batch, KV head) unit sharding used by
bench.py for multi-GPU runs: each rank computes its units (CPU oracle stands in for the
kernel), the unit buffers are all-gathered, and the result must equal the unsharded
computation bitwise."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_12798_b200.sharding import (gather_units, kv_head_shard, shard_views, unit_major,
                                            unit_shard)


@pytest.mark.parametrize("batch,hq,hkv", [(1, 32, 8), (2, 32, 8), (3, 6, 2), (5, 4, 4)])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_unit_plan_covers_every_batch_and_head(batch, hq, hkv, world):
    if world > batch * hkv:
        with pytest.raises(ValueError):
            unit_shard(0, world, batch, hq, hkv)
        return
    seen = []
    sizes = []
    for r in range(world):
        s = unit_shard(r, world, batch, hq, hkv)
        sizes.append(s.units)
        for b, kv0, kv1 in s.pieces:
            assert 0 <= kv0 < kv1 <= hkv
            seen += [(b, kv) for kv in range(kv0, kv1)]
    assert seen == [(b, kv) for b in range(batch) for kv in range(hkv)]  # each unit once, in order
    assert max(sizes) - min(sizes) <= 1  # balanced


def test_batch1_plan_is_kv_head_blocks():
    for world in (1, 2, 4, 8):
        for r in range(world):
            s = kv_head_shard(r, world, 32, 8)
            assert s.pieces == [(0, r * 8 // world, (r + 1) * 8 // world)]


def test_views_match_gqa_mapping():
    q = torch.arange(3 * 6 * 4 * 2).reshape(3, 6, 4, 2)
    k = torch.arange(3 * 2 * 4 * 2).reshape(3, 2, 4, 2)
    s = unit_shard(0, 2, 3, 6, 2)  # units [0, 3): (b0, kv0), (b0, kv1), (b1, kv0)
    assert s.pieces == [(0, 0, 2), (1, 0, 1)]
    (q0, k0, _), (q1, k1, _) = shard_views(q, k, k, s)
    assert torch.equal(q0, q[0:1, 0:6]) and torch.equal(k0, k[0:1, 0:2])
    assert torch.equal(q1, q[1:2, 0:3]) and torch.equal(k1, k[1:2, 0:1])
    assert unit_shard(1, 2, 3, 6, 2).pieces == [(1, 1, 2), (2, 0, 2)]
    assert torch.equal(unit_major(q, 2)[3], q[1, 3:6])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q, k, v, out_path):
    from oracle import vfa_oracle as vo
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B, Hq, L, d = q.shape
    sh = unit_shard(rank, world, B, Hq, k.shape[1])
    o_units = torch.empty((sh.units, sh.group, L, d), dtype=q.dtype)
    l_units = torch.empty((sh.units, sh.group, L), dtype=q.dtype)
    off = 0
    for qs, ks, vs in shard_views(q, k, v, sh):  # one launch per rectangular piece
        o, lse, _ = vo.forward(qs.numpy(), ks.numpy(), vs.numpy(), variant="vfa", causal=True,
                               q_block=32, k_block=32)
        n = ks.shape[1]
        o_units[off:off + n] = torch.from_numpy(o).reshape(n, sh.group, L, d)
        l_units[off:off + n] = torch.from_numpy(lse).reshape(n, sh.group, L)
        off += n
    o_all = gather_units(o_units, sh, world)
    l_all = gather_units(l_units, sh, world)
    if rank == 0:
        torch.save({"o": o_all.reshape(B, Hq, L, d), "lse": l_all.reshape(B, Hq, L)}, out_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("batch,hkv", [(1, 2), (3, 1)])
def test_gloo_world2_sharded_equals_unsharded(tmp_path, batch, hkv):
    # (3, 1): three units over two ranks -- uneven ranges, and rank 0's range spans two batch
    # entries (two launches), gathered with padding
    from oracle import vfa_oracle as vo
    g = torch.Generator().manual_seed(batch)
    q = torch.randn(batch, 4 * hkv, 128, 16, generator=g, dtype=torch.float64)
    k = torch.randn(batch, hkv, 128, 16, generator=g, dtype=torch.float64)
    v = torch.randn(batch, hkv, 128, 16, generator=g, dtype=torch.float64)
    out = str(tmp_path / "gathered.pt")
    mp.spawn(_worker, args=(2, _free_port(), q, k, v, out), nprocs=2, join=True)
    got = torch.load(out)
    ref_o, ref_lse, _ = vo.forward(q.numpy(), k.numpy(), v.numpy(), variant="vfa", causal=True,
                                   q_block=32, k_block=32)
    assert np.array_equal(got["o"].numpy(), ref_o)
    assert np.array_equal(got["lse"].numpy(), ref_lse)
