"""K10 (grouped tcgen05 FFN GEMM, optional SwiGLU epilogue) against a plain
PyTorch fp32 reference of the same op. Tolerance: one bf16 rounding of an
fp32-accumulated result (rtol 1e-2, atol 1e-2 on O(1) values)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(native_lib):
    return torch.device("cuda", 0)


def _rand(shape, dev, scale=1.0, seed=0):
    g = torch.Generator(device=dev).manual_seed(seed)
    return (torch.randn(shape, generator=g, device=dev) * scale).to(torch.bfloat16)


@pytest.mark.parametrize("M,K,N", [(1, 64, 32), (1000, 256, 768), (333, 4096, 1408), (4096, 1408, 2048)])
def test_dense_gemm_vs_fp32(dev, M, K, N):
    from paper_2601_06562_b200 import hotpath

    a = _rand((M, K), dev, seed=M)
    w = _rand((K, N), dev, 0.05, seed=N)
    out = torch.full((M, N), 7.0, device=dev).bfloat16()
    hotpath.ffn_gemm(a, w.t().contiguous(), out, N, m_host=M)
    ref = (a.float() @ w.float()).bfloat16().float()
    torch.testing.assert_close(out.float(), ref, rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("M,K,Fd", [(7, 256, 128), (2048, 256, 768), (1000, 2048, 1408)])
def test_dense_swiglu_vs_fp32(dev, M, K, Fd):
    from paper_2601_06562_b200 import hotpath

    x = _rand((M, K), dev, seed=1)
    wg = _rand((K, Fd), dev, 0.05, seed=2)
    wu = _rand((K, Fd), dev, 0.05, seed=3)
    out = torch.zeros((M, Fd), device=dev).bfloat16()
    hotpath.ffn_gemm(x, hotpath.interleave_gate_up(wg, wu), out, 2 * Fd, m_host=M, swiglu=True)
    ref = (F.silu(x.float() @ wg.float()) * (x.float() @ wu.float())).bfloat16().float()
    torch.testing.assert_close(out.float(), ref, rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("swiglu", [False, True])
def test_grouped_segments_with_empty_groups(dev, swiglu):
    """Groups of ragged (and empty) row segments, device offsets, each group
    with its own weights; rows outside every segment stay untouched."""
    from paper_2601_06562_b200 import hotpath

    rng = np.random.default_rng(4)
    G, K, Fd = 9, 512, 256
    counts = rng.integers(0, 300, size=G)
    counts[[1, 5]] = 0
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    P = int(off[-1])
    x = _rand((P + 40, K), dev, seed=5)
    wg = _rand((G, K, Fd), dev, 0.05, seed=6)
    wu = _rand((G, K, Fd), dev, 0.05, seed=7)
    n = 2 * Fd if swiglu else Fd
    w = hotpath.interleave_gate_up(wg, wu) if swiglu else wg.transpose(1, 2).contiguous()
    out = torch.full((P + 40, Fd), 3.0, device=dev).bfloat16()
    hotpath.ffn_gemm(x, w.view(G * n, K), out, n, group_off=torch.from_numpy(off).to(dev), groups=G, swiglu=swiglu)
    for g in range(G):
        a, b = int(off[g]), int(off[g + 1])
        if a == b:
            continue
        xg = x[a:b].float()
        ref = F.silu(xg @ wg[g].float()) * (xg @ wu[g].float()) if swiglu else xg @ wg[g].float()
        torch.testing.assert_close(out[a:b].float(), ref.bfloat16().float(), rtol=2e-2, atol=2e-2)
    assert torch.all(out[P:].float() == 3.0)


def test_grouped_from_moe_routing(dev):
    """K8's expert offsets drive K10 directly (no host round trip)."""
    from paper_2601_06562_b200 import hotpath

    rows, E, k, d, Fd = 3000, 16, 4, 256, 128
    logits = torch.randn(rows, E, device=dev)
    n = rows * k
    rrow = torch.empty(n, dtype=torch.int32, device=dev)
    rpos = torch.empty(n, dtype=torch.int32, device=dev)
    rw = torch.empty(n, device=dev)
    off = torch.empty(E + 1, dtype=torch.int32, device=dev)
    sc = torch.empty(hotpath.moe_route_scratch_bytes(rows, E), dtype=torch.uint8, device=dev)
    hotpath.moe_route(logits, k, rrow, rpos, rw, off, sc)
    h = _rand((rows, d), dev, seed=9)
    xin = torch.empty(n, d, device=dev).bfloat16()
    hotpath.gather_rows(h, rrow, xin, m_host=n)
    wg = _rand((E, d, Fd), dev, 0.05, seed=10)
    wu = _rand((E, d, Fd), dev, 0.05, seed=11)
    act = torch.empty(n, Fd, device=dev).bfloat16()
    hotpath.ffn_gemm(xin, hotpath.interleave_gate_up(wg, wu).view(E * 2 * Fd, d), act, 2 * Fd, group_off=off,
                     groups=E, swiglu=True)
    o = off.cpu().tolist()
    for e in range(E):
        xe = xin[o[e]:o[e + 1]].float()
        ref = (F.silu(xe @ wg[e].float()) * (xe @ wu[e].float())).bfloat16().float()
        torch.testing.assert_close(act[o[e]:o[e + 1]].float(), ref, rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("L,H,dh,theta,fused", [(1, 4, 64, 500000.0, False), (2048, 4, 64, 500000.0, False),
                                                (5000, 32, 128, 1e6, False), (3001, 28, 128, 1e6, True),
                                                (77, 3, 32, 1e4, True)])
def test_rope_vs_torch(dev, L, H, dh, theta, fused):
    """K11 rotary embedding of q and k in place against the torch fp32
    restatement (tests/torch_reference.py): one bf16 rounding apart at most.
    Head counts that are not a multiple of K11's 8-head chunk (Dream's 28),
    and q/k as strided views of one fused [L, 3*H*dh] qkv row."""
    from torch_reference import rope

    from paper_2601_06562_b200 import hotpath

    if fused:
        qkv = _rand((L, 3 * H * dh), dev, seed=7)
        v0 = qkv[:, 2 * H * dh:].clone()
        q, k = qkv[:, :H * dh], qkv[:, H * dh:2 * H * dh]
    else:
        q = _rand((L, H * dh), dev, seed=5)
        k = _rand((L, H * dh), dev, seed=6)
    inv = hotpath.rope_inv_freq(dh, theta, dev)
    rq, rk = rope(q, H, inv), rope(k, H, inv)
    hotpath.rope_qk_(q, k, H, inv)
    for got, want in ((q, rq), (k, rk)):
        torch.testing.assert_close(got.float(), want.float(), rtol=1e-2, atol=1e-2)
        assert (got != want).float().mean().item() < 0.01  # almost everywhere bit-equal
    if fused:
        assert torch.equal(qkv[:, 2 * H * dh:], v0)  # v untouched


@pytest.mark.parametrize("M,K,N", [(1, 128, 256), (777, 768, 256), (3000, 1408, 2048), (4096, 18944, 3584)])
def test_residual_epilogue_vs_fp32(dev, M, K, N):
    """K10 residual mode (the dense chunk's down projection + chunk write +
    residual add): out = bf16(out + a @ w) in place, one rounding of the fp32
    sum, against fp32 torch; rows past M untouched."""
    from paper_2601_06562_b200 import hotpath

    a = _rand((M, K), dev, seed=K)
    w = _rand((K, N), dev, 0.02, seed=N)
    res = _rand((M + 5, N), dev, seed=M)
    out = res.clone()
    hotpath.ffn_gemm(a, w.t().contiguous(), out[:M], N, m_host=M, residual=True)
    ref = (res[:M].float() + a.float() @ w.float()).bfloat16().float()
    torch.testing.assert_close(out[:M].float(), ref, rtol=1e-2, atol=1e-2)
    assert torch.equal(out[M:], res[M:])


@pytest.mark.parametrize("M,K,N,mode,groups", [(5000, 1024, 3072, "swiglu", 1), (4096, 2048, 512, "residual", 1),
                                               (777, 768, 256, "store", 1), (3000, 512, 1024, "swiglu", 4),
                                               (100, 256, 512, "store", 1)])
def test_k10_dynamic_schedule_bit_identical(dev, M, K, N, mode, groups):
    """K10 with the dynamic tile schedule (tiles claimed from a counter in the
    sched scratch, published through the unit ring) equals the static order
    bit for bit in every epilogue, dense and grouped; every tile claimed once."""
    from paper_2601_06562_b200 import hotpath

    a = _rand((M, K), dev, seed=11)
    w = _rand((groups * N, K), dev, scale=0.05, seed=12)
    off = None
    if groups > 1:
        cuts = sorted(np.random.default_rng(1).integers(0, M, groups - 1).tolist())
        off = torch.tensor([0] + cuts + [M], dtype=torch.int32, device=dev)
    base = _rand((M, N // 2 if mode == "swiglu" else N), dev, seed=13)
    outs = []
    for sched in (None, torch.full((4,), 9, dtype=torch.int32, device=dev)):
        out = base.clone()
        hotpath.ffn_gemm(a, w, out, N, group_off=off, groups=groups, m_host=M, swiglu=mode == "swiglu",
                         residual=mode == "residual", sched=sched)
        torch.cuda.synchronize()
        outs.append(out)
        if sched is not None:
            rows_blk = 256 if M > 128 else 128
            if off is None:
                tiles = -(-M // rows_blk) * -(-N // 256)
            else:
                o = off.cpu().tolist()
                tiles = sum(-(-(o[g + 1] - o[g]) // rows_blk) for g in range(groups)) * -(-N // 256)
            cg = 2 if M > 128 else 1
            units_cap = (-(-M // rows_blk) + groups) * -(-N // 256)  # the launch's grid bound (csrc/ffn_gemm.cu)
            workers = torch.cuda.get_device_properties(dev).multi_processor_count // cg
            pairs = min(units_cap, workers)
            if units_cap <= 2 * workers:  # small launches keep the static order: counters untouched
                assert int(sched[1]) == 9
            else:
                assert int(sched[1]) == tiles + pairs  # every tile claimed once, one failed claim per pair
    assert torch.equal(outs[0], outs[1])
