"""Host-side argument validation of the device wrappers (no GPU needed): the
wrappers reject malformed inputs with the reference's InputError
(mosaic/errors.py:41-42) before any launch, as the reference operator does
(mosaic/kernel.py:33-49)."""
import pytest
import torch

from paper_2601_06562_b200 import hotpath
from paper_2601_06562_b200.errors import InputError


def test_wrappers_reject_host_tensors_and_bad_dtypes():
    cpu_i32 = torch.zeros(16, dtype=torch.int32)
    with pytest.raises(InputError):
        hotpath.mask_compact(cpu_i32, 3, cpu_i32, cpu_i32[:1], torch.zeros(64, dtype=torch.uint8))
    with pytest.raises(InputError):
        hotpath.gather_rows(torch.zeros(4, 8), cpu_i32, torch.zeros(4, 8))
    with pytest.raises(InputError):
        hotpath.lmhead_stats(torch.zeros(4, 64, dtype=torch.bfloat16), torch.zeros(8, 64, dtype=torch.bfloat16),
                             1, torch.zeros(4), torch.zeros(4), torch.zeros(4, dtype=torch.int32))
    with pytest.raises(InputError):
        hotpath.swiglu_(torch.zeros(8, dtype=torch.bfloat16), torch.zeros(8, dtype=torch.bfloat16))
    with pytest.raises(InputError):
        hotpath.moe_route(torch.zeros(4, 8), 2, cpu_i32, cpu_i32, torch.zeros(16), cpu_i32,
                          torch.zeros(64, dtype=torch.uint8))
    with pytest.raises(InputError):
        hotpath.ffn_gemm(torch.zeros(4, 64), torch.zeros(32, 64, dtype=torch.bfloat16),
                         torch.zeros(4, 32, dtype=torch.bfloat16), 32)


def test_interleave_gate_up_layout():
    K, F = 3, 256
    g = torch.arange(K * F, dtype=torch.float32).view(K, F)
    u = -g
    w = hotpath.interleave_gate_up(g, u)
    assert w.shape == (2 * F, K)
    # block j: rows [256 j, 256 j + 128) = gate columns [128 j, 128 j + 128), then the matching up columns
    for j in range(F // 128):
        assert torch.equal(w[256 * j:256 * j + 128], g[:, 128 * j:128 * (j + 1)].t())
        assert torch.equal(w[256 * j + 128:256 * (j + 1)], u[:, 128 * j:128 * (j + 1)].t())
    with pytest.raises(InputError):
        hotpath.interleave_gate_up(torch.zeros(3, 100), torch.zeros(3, 100))
    # the executor's inverse restores the torch layout
    from torch_reference import _split_gate_up

    g2, u2 = _split_gate_up(w, F)
    assert torch.equal(g2, g) and torch.equal(u2, u)


def test_buffer_layout_alignment():
    lay = hotpath.BufferLayout()
    lay.add("a", (3,), torch.int32)
    lay.add("b", (5, 7), torch.bfloat16)
    lay.add("c", (1,), torch.float32)
    offs = [off for off, _, _ in lay.entries.values()]
    assert all(o % hotpath.ALIGN == 0 for o in offs) and offs == sorted(offs)
    views = lay.views(torch.zeros(lay.size, dtype=torch.uint8))
    assert views["b"].shape == (5, 7) and views["b"].dtype == torch.bfloat16
    with pytest.raises(InputError):
        lay.views(torch.zeros(lay.size - 1, dtype=torch.uint8))
