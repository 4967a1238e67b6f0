"""The reference operator's own test cases (pkg/tests/test_kernel.py) against
this package's drop-in `mosaic.kernel` API. Validation runs on the host (CPU
tests); the arithmetic cases run on the GPU through K2 + K3 with BF16
operands and FP32 accumulation, so the reference's 1e-12 float64 bound
becomes: exact where the operands are exactly representable in bf16 and the
sums in fp32 (the known-answer cases), and 1e-2 relative of the bf16-rounded
fp64 product otherwise (the reference's fp32-mode test uses 1e-5 on fp32
inputs; bf16 operands carry 2^-8 rounding)."""
import random

import numpy as np
import pytest
import torch

import mosaic_oracle as orc
from paper_2601_06562_b200 import GatherGemmProblem, gather_gemm, gemm_reference
from paper_2601_06562_b200.errors import InputError


# ----------------------------------------------------------------- host side (tests/test_kernel.py:87-97, :29-35)
def test_input_validation():
    hidden = np.zeros((4, 3))
    weight = np.zeros((3, 5))
    with pytest.raises(InputError):
        GatherGemmProblem(hidden, weight, (0, 0))  # duplicate index
    with pytest.raises(InputError):
        GatherGemmProblem(hidden, weight, (4,))  # out of range
    with pytest.raises(InputError):
        GatherGemmProblem(hidden, weight, (0,), tile_m=0)
    with pytest.raises(InputError):
        GatherGemmProblem(hidden, np.zeros((4, 5)), (0,))  # inner mismatch
    with pytest.raises(InputError):
        GatherGemmProblem(np.zeros(4), weight, (0,))  # not 2-D


def test_reference_examples():
    assert np.array_equal(gemm_reference([[2.0]], [[3.0]]), np.array([[6.0]]))
    assert np.array_equal(gemm_reference(np.zeros((2, 3)), np.zeros((3, 4))), np.zeros((2, 4)))
    with pytest.raises(InputError):
        gemm_reference(np.zeros((2, 3)), np.zeros((4, 4)))


# ----------------------------------------------------------------- device side
@pytest.mark.gpu
def test_identity_weight_selects_rows(native_lib):
    hidden = np.arange(12, dtype=np.float64).reshape(4, 3)
    out, _ = gather_gemm(GatherGemmProblem(hidden, np.eye(3), (2, 0)))
    assert np.array_equal(out, hidden[[2, 0], :])


@pytest.mark.gpu
def test_single_masked_row(native_lib):
    hidden = np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]])
    out, _ = gather_gemm(GatherGemmProblem(hidden, np.eye(2), (1,)))
    assert np.array_equal(out, np.array([[3.0, 4.0]]))


@pytest.mark.gpu
def test_random_problems_match_reference(native_lib):
    rng = random.Random(50)
    for _ in range(100):
        n, d, vocab = rng.randint(1, 9), rng.randint(1, 7), rng.randint(1, 11)
        hidden = np.array([[rng.uniform(-3, 3) for _ in range(d)] for _ in range(n)])
        weight = np.array([[rng.uniform(-3, 3) for _ in range(vocab)] for _ in range(d)])
        idx = tuple(rng.sample(range(n), rng.randint(1, n)))
        tiles = (rng.randint(1, 5), rng.randint(1, 5), rng.randint(1, 5))
        out, scratch = gather_gemm(GatherGemmProblem(hidden, weight, idx, *tiles))
        ref = gemm_reference(orc.bf16_round(hidden)[list(idx), :], orc.bf16_round(weight))
        assert np.allclose(out, ref, rtol=1e-5, atol=1e-5)  # fp32 accumulation of bf16 operands
        assert scratch.within_bound


@pytest.mark.gpu
def test_tile_size_invariance_is_bitwise(native_lib):
    rng = np.random.default_rng(51)
    hidden = rng.standard_normal((23, 17))
    weight = rng.standard_normal((17, 29))
    idx = tuple(int(i) for i in rng.choice(23, size=11, replace=False))
    outs = [gather_gemm(GatherGemmProblem(hidden, weight, idx, *t))[0]
            for t in ((1, 1, 1), (2, 5, 3), (7, 7, 7), (16, 4, 32), (64, 64, 64))]
    for other in outs[1:]:
        assert np.array_equal(outs[0], other)


@pytest.mark.gpu
def test_full_mask_reproduces_dense_product(native_lib):
    rng = np.random.default_rng(52)
    hidden = rng.standard_normal((13, 9))
    weight = rng.standard_normal((9, 21))
    idx = tuple(range(13))
    out, _ = gather_gemm(GatherGemmProblem(hidden, weight, idx))
    dense = orc.bf16_round(hidden) @ orc.bf16_round(weight)
    assert np.allclose(out, dense, rtol=1e-5, atol=1e-5)


@pytest.mark.gpu
def test_single_precision_mode(native_lib):
    rng = np.random.default_rng(53)
    hidden = rng.standard_normal((10, 6)).astype(np.float32)
    weight = rng.standard_normal((6, 8)).astype(np.float32)
    idx = (1, 4, 7)
    out, _ = gather_gemm(GatherGemmProblem(hidden, weight, idx))
    assert out.dtype == np.float32
    # exact up to fp32 accumulation on the bf16-rounded operands ...
    ref16 = gemm_reference(orc.bf16_round(hidden)[list(idx), :], orc.bf16_round(weight))
    assert np.allclose(out, ref16, rtol=1e-5, atol=1e-5)
    # ... and within the bf16 operand-rounding bound of the fp32 inputs' product
    ref = gemm_reference(hidden[list(idx), :], weight)
    bound = (np.abs(hidden[list(idx), :]) @ np.abs(weight)) * 2.0 ** -7
    assert np.all(np.abs(out.astype(np.float64) - ref) <= bound + 1e-6)


@pytest.mark.gpu
@pytest.mark.parametrize("layout,shift", [("dv", False), ("vd", True)])
def test_gather_logits_stats_sibling(native_lib, layout, shift):
    """The production sibling of gather_gemm: (token, lse, conf) per masked row,
    logits never materialised, against the oracle on the same bf16 operands."""
    from paper_2601_06562_b200 import gather_logits_stats

    rng = np.random.default_rng(9)
    n, d, V = 700, 256, 5000
    hidden = orc.bf16_round(rng.standard_normal((n, d)))
    w_dv = orc.bf16_round(rng.standard_normal((d, V)) * 0.05)
    idx = np.sort(rng.choice(n, 300, replace=False))
    weight = w_dv if layout == "dv" else np.ascontiguousarray(w_dv.T)
    tok, lse, conf = gather_logits_stats(hidden, weight, idx, weight_layout=layout, shift=shift)
    src = np.maximum(idx - 1, 0) if shift else idx
    ref = orc.softmax_stats(hidden[src] @ w_dv)
    ok = ref["margin"] > 1e-3
    assert np.array_equal(tok.cpu().numpy()[ok], ref["arg"][ok])
    assert orc.isclose_rel(lse.cpu().numpy(), ref["lse"], 1e-3)
    assert orc.isclose_rel(conf.cpu().numpy(), ref["conf"], 1e-3)


def test_scratch_account_is_a_real_bound(native_lib):
    """ScratchAccount (mosaic/kernel.py:52-59): the device account is the
    launched K3 configuration's on-chip staging per CTA, bounded by what one SM
    holds. It fails exactly where the reference's would: a global [m, d]
    gathered copy (the buffered K2 path), or a configuration larger than the
    SM. Host-only query, no kernel launch."""
    from paper_2601_06562_b200 import hotpath
    from paper_2601_06562_b200.kernel import SM_SMEM_OPTIN_BYTES, device_scratch

    for m, cg in ((16384, 2), (100, 1)):
        cfg = hotpath.lmhead_config(m, gather=True)
        assert cfg["cta_group"] == cg and cfg["a_rows"] == 128 and cfg["k_step"] == 64
        assert cfg["w_rows"] == 256 // cg and cfg["tmem_cols"] == 512
        assert cfg["smem_bytes"] <= SM_SMEM_OPTIN_BYTES
        staged = cfg["stages"] * (cfg["a_rows"] + cfg["w_rows"]) * cfg["k_step"]
        assert 2 * staged <= cfg["smem_bytes"]  # the panels are what the shared memory holds
        acc = device_scratch(m, 4096, gather=True)
        assert acc.peak_elements == staged + 128 * 512 and acc.within_bound
        assert not device_scratch(m, 4096, gather=False).within_bound  # a [m, d] copy breaks the bound
        assert not device_scratch(m, 4096, gather=True, smem_capacity_bytes=96 << 10).within_bound
