"""Seeded fuzz of the whole fused step against the oracle: random sequence
lengths, widths (multiples of 64), vocabulary sizes (ragged against the
256-column tile), mask densities and layouts, unmask counts, token shift,
and every K3 variant (runs mode, buffered or gather mode, default or
die-aware unit schedule, single-SM or pair tiles), and temperature sampling in a third of the
buffered cases. Tolerances as tests/test_gpu_parity.py:
indices and selections bit-exact, tokens exact where the fp64 top-1 margin
exceeds 1e-3, lse / confidence within 1e-3 relative.
"""
import os

import numpy as np
import pytest
import torch

import mosaic_oracle as orc

pytestmark = pytest.mark.gpu

N_CASES = int(os.environ.get("MOSAIC_FUZZ_CASES", "48"))


@pytest.fixture(scope="module")
def dev(native_lib):
    return torch.device("cuda", 0)


def _case(i: int):
    rng = np.random.default_rng(1000 + i)
    L = int(rng.integers(1, 6000))
    d = int(64 * rng.integers(1, 17))
    V = int(rng.integers(2, 20000))
    density = float(rng.choice([0.0, 0.01, 0.3, 0.5, 0.9, 1.0]))
    layout = str(rng.choice(["scattered", "suffix", "blocks"]))
    k = int(rng.integers(0, 300))
    shift = bool(rng.integers(0, 2))
    a_path = str(rng.choice(["runs", "buffered", "gather"]))  # K3's A operand: runs mode (default) / K2 all / H
    die = bool(rng.integers(0, 2))
    temperature = float(rng.choice([0.0, 0.0, 0.5, 1.5])) if a_path != "gather" else 0.0  # sampling: buffered A
    return rng, L, d, V, density, layout, k, shift, a_path, die, temperature


@pytest.mark.parametrize("i", range(N_CASES))
def test_fused_step_fuzz(dev, i):
    from paper_2601_06562_b200 import MaskOnlyHead

    rng, L, d, V, density, layout, k, shift, a_path, die, temperature = _case(i)
    mask_id = V - 1
    x = rng.integers(0, max(V - 1, 1), size=L).astype(np.int32)
    if layout == "scattered":
        x[rng.random(L) < density] = mask_id
    elif layout == "suffix":
        x[L - int(round(density * L)):] = mask_id
    else:  # a few masked blocks
        for _ in range(int(rng.integers(1, 5))):
            a = int(rng.integers(0, L))
            x[a:a + int(density * L / 3) + 1] = mask_id
    H = orc.bf16_round(rng.standard_normal((L, d)))
    W = orc.bf16_round(rng.standard_normal((V, d)) * float(rng.choice([0.02, 0.1])))
    Hd = torch.from_numpy(H.astype(np.float32)).to(dev).bfloat16()
    Wd = torch.from_numpy(W.astype(np.float32)).to(dev).bfloat16()
    head = MaskOnlyHead(Wd, seq_len=L, mask_id=mask_id, shift=shift, fused_gather=a_path == "gather",
                        die_aware=die, temperature=temperature, seed=i)
    if a_path == "buffered":
        head.a_runs = False
    xd = torch.from_numpy(x).to(dev)
    out = head.step(xd, Hd, k)
    torch.cuda.synchronize()
    ref = orc.step(x, H, W, mask_id, k, shift=shift)
    if temperature > 0:  # Gumbel-max sample with the head's first-step seed, noise keyed by position
        idx = ref["idx"]
        src = np.maximum(idx - 1, 0) if shift else idx
        seed0 = (i * 0x9E3779B1 + 0x27D4EB2F) & 0xFFFFFFFF
        smp = orc.sample_stats(orc.logits_f64(H[src], W), idx, seed0, temperature)
        ref = dict(ref, arg=smp["arg"], conf=smp["conf"], margin=smp["margin"])
        ref["selected"] = orc.remask_select(smp["conf"], idx, k)
    M = int(out.m_dev.item())
    assert M == ref["idx"].size
    assert np.array_equal(out.idx[:M].cpu().numpy(), ref["idx"])
    xo = xd.cpu().numpy()
    if M == 0:
        assert np.array_equal(xo, x)
        return
    token = out.token[:M].cpu().numpy()
    ok = ref["margin"] > 1e-3
    assert np.array_equal(token[ok], ref["arg"][ok])
    assert orc.isclose_rel(out.lse[:M].cpu().numpy().astype(np.float64), ref["lse"], 1e-3)
    # sampled rows whose noisy top-2 are within the margin may pick another token, and with it another p(token)
    rows = ok if temperature > 0 else np.ones(M, dtype=bool)
    assert orc.isclose_rel(out.conf[:M].cpu().numpy().astype(np.float64)[rows], ref["conf"][rows], 1e-3)
    sel = out.selected[:M].cpu().numpy().astype(bool)
    assert np.array_equal(sel, orc.remask_select(out.conf[:M].cpu().numpy(), ref["idx"], k))
    if rows.all():
        near = orc.near_tie_rows(ref["conf"], k)
        assert np.array_equal(sel[~near], ref["selected"][~near])
    assert int(sel.sum()) == min(k, M)
    # untouched outside the committed rows; committed rows carry the device token
    changed = np.flatnonzero(xo != x)
    committed = ref["idx"][sel]
    assert set(changed.tolist()) <= set(committed.tolist())
    assert np.array_equal(xo[committed], token[sel])
