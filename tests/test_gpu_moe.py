"""MoE expert FFN (BASELINE configs[3]) on the GPU: K8 routing and K9 combine
against the CPU oracle through the C ABI, and the chunked expert FFN executed
inside the cuMem arena against a plain-PyTorch forward of the same model.

Tolerances: dispatch order, combine positions and expert offsets bit-exact;
routing weights within 1e-6 relative (fp32 softmax); combine within one bf16
ulp of the fp64 oracle; the in-arena forward within 2e-2 of plain PyTorch (the
dense executor test's bf16 tolerance).
"""
from dataclasses import replace

import numpy as np
import pytest
import torch

import mosaic_oracle as orc

pytestmark = pytest.mark.gpu

MASK_ID = 8191


@pytest.fixture(scope="module")
def dev(native_lib):
    return torch.device("cuda", 0)


def _route(logits_np, k, dev, row_base=0):
    from paper_2601_06562_b200 import hotpath

    rows, E = logits_np.shape
    z = torch.from_numpy(logits_np.astype(np.float32)).to(dev)
    n = max(rows * k, 1)
    drow = torch.full((n,), -1, dtype=torch.int32, device=dev)
    pos = torch.full((n,), -1, dtype=torch.int32, device=dev)
    w = torch.zeros(n, dtype=torch.float32, device=dev)
    off = torch.full((E + 1,), -1, dtype=torch.int32, device=dev)
    scratch = torch.empty(hotpath.moe_route_scratch_bytes(rows, E), dtype=torch.uint8, device=dev)
    hotpath.moe_route(z, k, drow, pos, w, off, scratch, row_base=row_base)
    return drow.cpu().numpy()[: rows * k], pos.cpu().numpy()[: rows * k], w.cpu().numpy()[: rows * k], off.cpu().numpy()


@pytest.mark.parametrize("rows,E,k,ties", [(1, 4, 1, False), (37, 8, 2, False), (1000, 64, 8, False),
                                           (4099, 64, 8, True), (65536, 64, 8, False), (300, 256, 16, True),
                                           (129, 7, 7, True)])
def test_route_vs_oracle(dev, rows, E, k, ties):
    rng = np.random.default_rng(rows + E)
    z = rng.standard_normal((rows, E)).astype(np.float32)
    if ties:  # integer logits: many exact ties, broken by expert id
        z = rng.integers(-2, 3, size=(rows, E)).astype(np.float32)
    drow, pos, w, off = _route(z, k, dev, row_base=5)
    ref = orc.moe_route(z, k, row_base=5)
    assert np.array_equal(off, ref["expert_off"])
    assert np.array_equal(drow, ref["disp_row"])
    assert np.array_equal(pos, ref["comb_pos"].reshape(-1))
    assert orc.isclose_rel(w, ref["comb_w"].reshape(-1), 1e-6)


def test_route_empty(dev):
    from paper_2601_06562_b200 import hotpath

    off = torch.full((9,), -1, dtype=torch.int32, device=dev)
    e = torch.empty(0, dtype=torch.int32, device=dev)
    hotpath.moe_route(torch.empty((0, 8), dtype=torch.float32, device=dev), 2, e, e,
                      torch.empty(0, dtype=torch.float32, device=dev), off,
                      torch.empty(256, dtype=torch.uint8, device=dev))
    assert off.cpu().tolist() == [0] * 9


def test_route_rejects_bad_args(dev):
    from paper_2601_06562_b200 import hotpath
    from paper_2601_06562_b200.errors import InputError

    z = torch.zeros((4, 300), dtype=torch.float32, device=dev)
    buf = torch.zeros(4096, dtype=torch.int32, device=dev)
    with pytest.raises(InputError):
        hotpath.moe_route(z, 2, buf, buf, buf.view(torch.float32), buf, buf.view(torch.uint8))


@pytest.mark.parametrize("rows,k,d", [(1, 1, 8), (513, 2, 256), (4096, 8, 2048)])
def test_combine_vs_oracle(dev, rows, k, d):
    from paper_2601_06562_b200 import hotpath

    rng = np.random.default_rng(rows * k)
    src = orc.bf16_round(rng.standard_normal((rows * k, d)))
    pos = rng.permutation(rows * k).reshape(rows, k).astype(np.int32)
    w = rng.random((rows, k)).astype(np.float32)
    out = torch.empty((rows, d), dtype=torch.bfloat16, device=dev)
    hotpath.moe_combine(torch.from_numpy(src.astype(np.float32)).to(dev).bfloat16(),
                        torch.from_numpy(pos.reshape(-1)).to(dev), torch.from_numpy(w.reshape(-1)).to(dev), k, out)
    ref = orc.moe_combine(src, pos, w.astype(np.float64))
    got = out.float().cpu().numpy()
    # one bf16 rounding of an fp32 sum: <= 2^-8 relative (+ tiny absolute)
    assert np.all(np.abs(got - ref) <= 2.0 ** -8 * np.abs(ref) + 1e-6)


# ----------------------------------------------------------------- executor
@pytest.fixture(scope="module")
def env(dev):
    from paper_2601_06562_b200 import vmm, workload
    from paper_2601_06562_b200.executor import RandomDLLM, StepExecutor

    cfg = workload.toy_configs()["tiny_moe"]
    model = RandomDLLM(cfg, dev, seed=11)
    ws = vmm.reserve(8 << 30, backend="cuda")
    ex = StepExecutor(model, ws, MASK_ID)
    yield cfg, model, ex
    ws.close()


def _x(L, n_masked, dev, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.integers(0, MASK_ID, size=L).astype(np.int32)
    x[L - n_masked:] = MASK_ID
    return torch.from_numpy(x).to(dev)


@pytest.mark.parametrize("K_ffn", [1, 3, 7])
def test_moe_forward_in_arena_matches_plain_torch(env, dev, K_ffn):
    from torch_reference import reference_forward

    cfg, model, ex = env
    L, M = 2048, 1024
    x = _x(L, M, dev)
    ref_h = reference_forward(model, x.clone())
    g = ex_graph(cfg, L, M, (1, K_ffn))
    out = ex.run(g, x.clone(), 0, keep=("l1.h_out",))
    h = out["kept"]["l1.h_out"].float()
    assert torch.isfinite(h).all()
    torch.testing.assert_close(h, ref_h.float(), rtol=2e-2, atol=2e-2)
    assert out["committed_bytes"] >= out["workspace_bytes"]  # the arena only grows across steps


def ex_graph(cfg, L, M, K):
    from paper_2601_06562_b200 import workload

    t = workload.build_layer_template(cfg)
    return t.instantiate({"L": L, "M": M, "K_logits": K[0], "K_FFN": K[1]})


@pytest.mark.parametrize("mode", ["fused", "fused_gather"])
def test_moe_fused_step_vs_oracle(env, dev, mode):
    """The hot path (K1-K5, or K1 + gather-mode K3 + K4/K5) after the in-arena
    MoE forward, checked against the CPU oracle on the executor's own final
    hidden states."""
    cfg, model, ex = env
    L, M, k = 2048, 1024, 64
    x = _x(L, M, dev, seed=4)
    x0 = x.cpu().numpy()
    out = ex.run(ex_graph(replace(cfg, logits_mode=mode), L, M, (2, 3)), x, k, keep=("l1.h_out", "token_out"))
    h = out["kept"]["l1.h_out"].float().cpu().numpy().astype(np.float64)
    ref = orc.step(x0, h, model.w_vocab.float().cpu().numpy().astype(np.float64), MASK_ID, k)
    tok = out["kept"]["token_out"].cpu().numpy()
    conf = out["kept"]["confidence"].cpu().numpy()
    ok = ref["margin"] > 1e-3
    assert np.array_equal(tok[ok], ref["arg"][ok])
    assert orc.isclose_rel(conf, ref["conf"], 1e-3)
    sel = (x.cpu().numpy() != MASK_ID)[ref["idx"]]
    assert sel.sum() == k
    assert np.array_equal(sel, orc.remask_select(conf, ref["idx"], k))
