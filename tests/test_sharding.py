"""Multi-process (gloo, world size 2) test of the KV-head sharding used by bench.py for
multi-GPU runs: each rank computes its shard (CPU oracle stands in for the kernel), the
shards are all-gathered, and the result must equal the unsharded computation bitwise."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_12798_b200.sharding import gather_heads, kv_head_shard, shard_inputs


def test_shard_plan_covers_all_heads():
    for world in (1, 2, 4, 8):
        seen_q, seen_kv = [], []
        for r in range(world):
            s = kv_head_shard(r, world, 32, 8)
            seen_q += list(range(s.q0, s.q1))
            seen_kv += list(range(s.kv0, s.kv1))
            assert (s.q1 - s.q0) == 4 * (s.kv1 - s.kv0)
            assert s.q0 // 4 == s.kv0  # GQA mapping h // (Hq/Hkv) stays inside the shard
        assert seen_q == list(range(32)) and seen_kv == list(range(8))
    with pytest.raises(ValueError):
        kv_head_shard(0, 3, 32, 8)


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
    sh = kv_head_shard(rank, world, q.shape[1], k.shape[1])
    qs, ks, vs = shard_inputs(q, k, v, sh)
    o, lse, _ = vo.forward(qs.numpy(), ks.numpy(), vs.numpy(), variant="vfa", causal=True,
                           q_block=32, k_block=32)
    o_all = gather_heads(torch.from_numpy(o), world)
    l_all = gather_heads(torch.from_numpy(lse), world)
    if rank == 0:
        torch.save({"o": o_all, "lse": l_all}, out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharded_equals_unsharded(tmp_path):
    from oracle import vfa_oracle as vo
    g = torch.Generator().manual_seed(0)
    q = torch.randn(1, 8, 128, 16, generator=g, dtype=torch.float64)
    k = torch.randn(1, 2, 128, 16, generator=g, dtype=torch.float64)
    v = torch.randn(1, 2, 128, 16, generator=g, dtype=torch.float64)
    out = str(tmp_path / "gathered.pt")
    mp.spawn(_worker, args=(2, _free_port(), q, k, v, out), nprocs=2, join=True)
    got = torch.load(out)
    ref_o, ref_lse, _ = vo.forward(q.numpy(), k.numpy(), v.numpy(), variant="vfa", causal=True,
                                   q_block=32, k_block=32)
    assert np.array_equal(got["o"].numpy(), ref_o)
    assert np.array_equal(got["lse"].numpy(), ref_lse)
