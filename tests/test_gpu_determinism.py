"""Run-to-run determinism of every kernel family (the reference pins
byte-identical plans and replays, tests/test_planner.py:160-169,
tests/test_allocsim.py:157-161): the same inputs give bit-identical outputs
on repeated launches -- fixed split/rank merge order, no float atomics in any
reduction that feeds an output."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev(native_lib):
    return torch.device("cuda", 0)


def test_fused_step_bitwise_repeatable(dev):
    from paper_2601_06562_b200 import MaskOnlyHead

    g = torch.Generator(device=dev).manual_seed(0)
    L, d, V, mid, k = 8192, 1024, 50000, 49999, 300
    H = torch.randn(L, d, generator=g, device=dev).bfloat16()
    W = (torch.randn(V, d, generator=g, device=dev) * 0.03).bfloat16()
    x0 = torch.randint(0, V - 1, (L,), generator=g, device=dev, dtype=torch.int32)
    x0[torch.rand(L, generator=g, device=dev) < 0.5] = mid
    runs = []
    for fg in (False, False, True, True):
        head = MaskOnlyHead(W, seq_len=L, mask_id=mid, fused_gather=fg)
        x = x0.clone()
        o = head.step(x, H, k)
        torch.cuda.synchronize()
        M = int(o.m_dev.item())
        runs.append([t.cpu() for t in (x, o.token[:M], o.lse[:M], o.conf[:M], o.selected[:M])])
    for r in runs[1:]:
        for a, b in zip(runs[0], r):
            assert torch.equal(a, b)


def test_moe_and_ffn_kernels_bitwise_repeatable(dev):
    from paper_2601_06562_b200 import hotpath

    g = torch.Generator(device=dev).manual_seed(1)
    rows, E, k, d, f = 5000, 32, 4, 512, 256
    z = torch.randn(rows, E, generator=g, device=dev)
    h = torch.randn(rows, d, generator=g, device=dev).bfloat16()
    wgu = (torch.randn(E * 2 * f, d, generator=g, device=dev) * 0.05).bfloat16()
    wd = (torch.randn(E * d, f, generator=g, device=dev) * 0.05).bfloat16()
    outs = []
    for _ in range(2):
        n = rows * k
        rrow, rpos = (torch.empty(n, dtype=torch.int32, device=dev) for _ in range(2))
        rw, off = torch.empty(n, device=dev), torch.empty(E + 1, dtype=torch.int32, device=dev)
        hotpath.moe_route(z, k, rrow, rpos, rw, off,
                          torch.empty(hotpath.moe_route_scratch_bytes(rows, E), dtype=torch.uint8, device=dev))
        xin = torch.empty(n, d, device=dev).bfloat16()
        hotpath.gather_rows(h, rrow, xin, m_host=n)
        act = torch.empty(n, f, device=dev).bfloat16()
        hotpath.ffn_gemm(xin, wgu, act, 2 * f, group_off=off, groups=E, swiglu=True)
        down = torch.empty(n, d, device=dev).bfloat16()
        hotpath.ffn_gemm(act, wd, down, d, group_off=off, groups=E)
        y = torch.empty(rows, d, device=dev).bfloat16()
        hotpath.moe_combine(down, rpos, rw, k, y)
        torch.cuda.synchronize()
        outs.append([t.cpu() for t in (rrow, rpos, rw, off, act, down, y)])
    for a, b in zip(*outs):
        assert torch.equal(a, b)
