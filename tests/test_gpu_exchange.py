"""K4x, the vocab-shard exchange over peer memory (csrc/exchange.cu), on one
B200: (1) a real NCCL process group of world 1 -- push/wait/merge through the
symmetric buffers equals the ungrouped step bit for bit; (2) two processes
sharing the GPU (gloo group; symmetric memory mapped across the processes
with CUDA IPC, the same peer-pointer path NVLink peers use), each holding half
of the vocab: both ranks commit exactly what the unsharded step commits."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(dev, seed=7):
    rng = np.random.default_rng(seed)
    L, d, V, mask_id, k = 4096, 512, 16384, 16383, 100
    x = rng.integers(0, V - 1, size=L).astype(np.int32)
    x[rng.random(L) < 0.5] = mask_id
    H = torch.from_numpy(rng.standard_normal((L, d)).astype(np.float32)).to(dev).bfloat16()
    W = torch.from_numpy((rng.standard_normal((V, d)) * 0.05).astype(np.float32)).to(dev).bfloat16()
    return L, V, mask_id, k, x, H, W


def test_p2p_exchange_world1(native_lib):
    import torch.distributed as dist

    from paper_2601_06562_b200 import MaskOnlyHead

    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0, world_size=1, device_id=dev)
    try:
        L, V, mask_id, k, x, H, W = _problem(dev)
        outs = []
        for kw in ({}, {"group": dist.group.WORLD, "exchange": "p2p"}):
            head = MaskOnlyHead(W, seq_len=L, mask_id=mask_id, **kw)
            for _ in range(3):  # several epochs through the same signal pads
                xd = torch.from_numpy(x).to(dev)
                o = head.step(xd, H, k)
            torch.cuda.synchronize()
            M = int(o.m_dev.item())
            outs.append((xd.cpu(), o.token[:M].cpu(), o.lse[:M].cpu(), o.conf[:M].cpu()))
        for a, b in zip(*outs):
            assert torch.equal(a, b)
    finally:
        dist.destroy_process_group()


def _rank_main(rank, world, bufs, q, delay=0.0):
    """One vocab shard; peers reached through CUDA-IPC mappings of the other
    process's gathered/signal buffers (what symmetric memory provides across
    NVLink peers). ``delay`` > 0: rank 1's host sleeps between enqueuing its
    push and its wait, so the peer finishes its wait, runs a whole step and
    publishes the next epoch before this rank's wait of the current one runs
    (the case a wait for "slot == epoch" would miss)."""
    import sys
    import time

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2601_06562_b200 import MaskOnlyHead, shard

    try:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        gathered, signal = bufs
        ex = shard.P2PExchange.from_buffers(gathered[rank], signal[rank], [g.data_ptr() for g in gathered],
                                            [t.data_ptr() for t in signal], rank, world)
        L, V, mask_id, k, x, H, W = _problem(dev)
        v0, v1 = shard.vocab_shard_bounds(V, world, rank)
        head = MaskOnlyHead(W[v0:v1].contiguous(), seq_len=L, mask_id=mask_id, vocab_offset=v0, m_cap=L,
                            exchange=ex)
        if delay > 0 and rank == 1:
            wait = ex.wait

            def late_wait(stream=None):
                torch.cuda.synchronize()  # this rank's push has landed; the peer can run ahead
                time.sleep(delay)
                wait(stream)

            ex.wait = late_wait
        for _ in range(3):  # three epochs through the same pads
            xd = torch.from_numpy(x).to(dev)
            o = head.step(xd, H, k)
        torch.cuda.synchronize()
        M = int(o.m_dev.item())
        q.put((rank, xd.cpu().numpy(), o.token[:M].cpu().numpy(), o.conf[:M].cpu().numpy()))
        del ex, head, gathered, signal, bufs  # release the IPC mappings before the producer goes away
        torch.cuda.synchronize()
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, "error", repr(exc), None))


@pytest.mark.parametrize("delay", [0.0, 0.5])
def test_p2p_exchange_two_ranks_one_gpu(native_lib, delay):
    import torch.multiprocessing as mp

    from paper_2601_06562_b200 import MaskOnlyHead

    dev = torch.device("cuda", 0)
    L, V, mask_id, k, x, H, W = _problem(dev)
    world = 2
    gathered = [torch.zeros(2, world, 3, L, device=dev) for _ in range(world)]
    signal = [torch.zeros(world, dtype=torch.int32, device=dev) for _ in range(world)]
    torch.cuda.synchronize()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, world, (gathered, signal), q, delay)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in procs:
        r, a, b, c = q.get(timeout=300)
        res[r] = (a, b, c)
    for p in procs:
        p.join(timeout=120)
    errors = [v[1] for v in res.values() if isinstance(v[0], str)]
    assert not errors, errors
    ref_head = MaskOnlyHead(W, seq_len=L, mask_id=mask_id)
    xd = torch.from_numpy(x).to(dev)
    o = ref_head.step(xd, H, k)
    torch.cuda.synchronize()
    M = int(o.m_dev.item())
    for r in range(world):
        xo, tok, conf = res[r]
        assert np.array_equal(xo, xd.cpu().numpy())       # identical commits on every rank
        assert np.array_equal(tok, o.token[:M].cpu().numpy())
        assert np.allclose(conf, o.conf[:M].cpu().numpy(), rtol=1e-5)  # rank-order merge vs split merge


def _exec_rank(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2601_06562_b200 import shard, vmm, workload
    from paper_2601_06562_b200.executor import RandomDLLM, StepExecutor

    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        cfg = workload.toy_configs()["tiny_llada"]
        model = RandomDLLM(cfg, dev, seed=3, vocab_shard=shard.vocab_shard_bounds(cfg.vocab_size, world, rank))
        ws = vmm.reserve(2 << 30, backend="cuda")
        ex = StepExecutor(model, ws, 8191, group=dist.group.WORLD)
        x = _exec_x(dev)
        g = workload.build_layer_template(cfg).instantiate({"L": 2048, "M": 1024, "K_logits": 2, "K_FFN": 2})
        ex.run(g, x, 64)
        torch.cuda.synchronize()
        q.put((rank, x.cpu().numpy()))
        ws.close()
    except Exception as exc:
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def _exec_x(dev):
    rng = np.random.default_rng(12)
    x = rng.integers(0, 8191, size=2048).astype(np.int32)
    x[1024:] = 8191
    return torch.from_numpy(x).to(dev)


def test_vocab_sharded_executor_two_ranks(native_lib):
    """The step executor with a vocab-sharded LM head on two ranks (gloo
    all-gather of the triples, both processes on this GPU): every rank commits
    what the unsharded executor commits."""
    import torch.multiprocessing as mp

    from paper_2601_06562_b200 import vmm, workload
    from paper_2601_06562_b200.executor import RandomDLLM, StepExecutor

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_exec_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    assert all(not isinstance(v, str) for v in res.values()), res
    dev = torch.device("cuda", 0)
    cfg = workload.toy_configs()["tiny_llada"]
    model = RandomDLLM(cfg, dev, seed=3)
    ws = vmm.reserve(2 << 30, backend="cuda")
    try:
        x = _exec_x(dev)
        g = workload.build_layer_template(cfg).instantiate({"L": 2048, "M": 1024, "K_logits": 2, "K_FFN": 2})
        StepExecutor(model, ws, 8191).run(g, x, 64)
        want = x.cpu().numpy()
    finally:
        ws.close()
    for r in (0, 1):
        assert np.array_equal(res[r], want)
