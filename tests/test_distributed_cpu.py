"""The N>1 (vocab-sharded) host path on CPU with world_size-2 gloo: shard
bounds, the triple exchange layout that K4 consumes, and the rank-order merge
that makes every rank reach the same tokens and remask selection."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import mosaic_oracle as orc
from paper_2601_06562_b200.shard import exchange_triples, pack_triples, unpack_triples, vocab_shard_bounds


def test_shard_bounds_partition_vocab():
    for V in (126464, 152064, 8192, 7):
        for P in (1, 2, 4, 8):
            b = [vocab_shard_bounds(V, P, r) for r in range(P)]
            assert b[0][0] == 0 and b[-1][1] == V
            assert all(b[i][1] == b[i + 1][0] for i in range(P - 1))
            assert max(e - s for s, e in b) - min(e - s for s, e in b) <= 1
    assert vocab_shard_bounds(126464, 8, 3) == (47424, 63232)  # 15808 per rank
    with pytest.raises(ValueError):
        vocab_shard_bounds(10, 2, 2)


def test_pack_roundtrip_keeps_argmax_bits():
    mx = torch.tensor([1.5, -2.0, 3.0])
    sm = torch.tensor([2.0, 4.0, 1.0])
    arg = torch.tensor([126463, 0, 2 ** 30], dtype=torch.int32)
    m2, s2, a2 = unpack_triples(pack_triples(mx, sm, arg))
    assert torch.equal(m2, mx) and torch.equal(s2, sm) and torch.equal(a2, arg)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, V, m, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(seed)
        z = rng.standard_normal((m, V)) * 2.0  # the same logits on every rank (replicated rows)
        v0, v1 = vocab_shard_bounds(V, world, rank)
        # this rank's K3+K4 result for its slice: one triple per row, global ids
        (mx, sm, arg), = orc.split_stats(z[:, v0:v1], [0, v1 - v0], v_offset=v0)
        local = pack_triples(torch.tensor(mx, dtype=torch.float32), torch.tensor(sm, dtype=torch.float32),
                             torch.tensor(arg, dtype=torch.int32))
        g = exchange_triples(local)
        assert g.shape == (world, 3, m)
        gm, gs, ga = unpack_triples(g)
        # K4's view of the gathered block: rank r's triple at offset r*3*m
        flat = g.view(-1)
        for r in range(world):
            assert torch.equal(flat[r * 3 * m: r * 3 * m + m], gm[r])
        parts = [(gm[r].double().numpy(), gs[r].double().numpy(), ga[r].numpy()) for r in range(world)]
        m_all, s_all, a_all = orc.merge_triples(parts)
        conf = 1.0 / s_all
        sel = orc.remask_select(conf.astype(np.float32), np.arange(m), m // 4)
        q.put((rank, a_all.tolist(), conf.tolist(), sel.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("V,m,world", [(1000, 64, 2), (126464 // 64, 33, 2), (1001, 40, 4)])
def test_vocab_sharded_merge_world2(V, m, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, V, m, 7, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        rank, a, c, s = q.get(timeout=120)
        res[rank] = (a, c, s)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # every rank reached the same tokens, confidences and selection ...
    assert all(res[r] == res[0] for r in range(world))
    # ... equal to the unsharded statistics
    z = np.random.default_rng(7).standard_normal((m, V)) * 2.0
    whole = orc.softmax_stats(z)
    assert res[0][0] == whole["arg"].tolist()
    assert np.allclose(res[0][1], whole["conf"], rtol=1e-6)
