"""The planned step executed on the GPU: every activation lives at its
first-fit offset inside one cuMem arena, the FFN and logits run as lazily
chunked loops, and the fused hot path (K1..K5) commits tokens. Checked
against a plain-PyTorch forward of the same random-init model and the CPU
oracle for the hot path."""
from dataclasses import replace

import numpy as np
import pytest
import torch

import mosaic_oracle as orc

pytestmark = pytest.mark.gpu

MASK_ID = 8191


@pytest.fixture(scope="module")
def env(native_lib):
    from paper_2601_06562_b200 import vmm, workload
    from paper_2601_06562_b200.executor import RandomDLLM, StepExecutor

    cfg = workload.toy_configs()["tiny_llada"]
    dev = torch.device("cuda", 0)
    model = RandomDLLM(cfg, dev, seed=3)
    ws = vmm.reserve(8 << 30, backend="cuda")
    ex = StepExecutor(model, ws, MASK_ID)
    yield cfg, model, ex, dev
    ws.close()


def _x(L, n_masked, dev, seed=0):
    rng = np.random.default_rng(seed)
    x = rng.integers(0, MASK_ID, size=L).astype(np.int32)
    x[L - n_masked:] = MASK_ID
    return torch.from_numpy(x).to(dev)


def _step(cfg, ex, x, M, k, K=(1, 1), mode="fused", keep=()):
    from paper_2601_06562_b200 import workload

    t = workload.build_layer_template(replace(cfg, logits_mode=mode))
    g = t.instantiate({"L": x.numel(), "M": M, "K_logits": K[0], "K_FFN": K[1]})
    return ex.run(g, x, k, keep=keep)


def test_forward_in_arena_matches_plain_torch(env):
    from torch_reference import reference_forward

    cfg, model, ex, dev = env
    L, M = 2048, 1024
    x = _x(L, M, dev)
    ref_h = reference_forward(model, x.clone())
    out = _step(cfg, ex, x.clone(), M, 0, keep=("l1.h_out",))
    h = out["kept"]["l1.h_out"]
    assert torch.isfinite(h.float()).all()
    torch.testing.assert_close(h.float(), ref_h.float(), rtol=2e-2, atol=2e-2)
    assert out["committed_bytes"] >= out["workspace_bytes"]
    assert out["committed_bytes"] - out["workspace_bytes"] < ex.ws.page_size


@pytest.mark.parametrize("K", [(1, 1), (3, 2), (7, 5)])
def test_fused_step_vs_oracle(env, K):
    cfg, model, ex, dev = env
    L, M, k = 2048, 1024, 64
    x = _x(L, M, dev, seed=1)
    x0 = x.cpu().numpy()
    out = _step(cfg, ex, x, M, k, K=K, keep=("l1.h_out", "token_out"))
    h = out["kept"]["l1.h_out"].float().cpu().numpy().astype(np.float64)
    W = model.w_vocab.float().cpu().numpy().astype(np.float64)
    ref = orc.step(x0, h, W, MASK_ID, k)
    tok = out["kept"]["token_out"].cpu().numpy()
    conf = out["kept"]["confidence"].cpu().numpy()
    ok = ref["margin"] > 1e-3
    assert np.array_equal(tok[ok], ref["arg"][ok])
    assert orc.isclose_rel(conf, ref["conf"], 1e-3)
    xo = x.cpu().numpy()
    sel_dev = (xo != MASK_ID)[ref["idx"]]
    assert sel_dev.sum() == k
    assert np.array_equal(sel_dev, orc.remask_select(conf, ref["idx"], k))
    near = orc.near_tie_rows(ref["conf"], k)
    assert np.array_equal(sel_dev[~near], ref["selected"][~near])


def test_modes_agree(env):
    """fused (K2-K5) vs the reference's materialising mask-only and eager modes."""
    cfg, model, ex, dev = env
    L, M, k = 2048, 1024, 32
    x0 = _x(L, M, dev, seed=2)
    outs = {}
    for mode in ("fused", "mask_only", "eager"):
        x = x0.clone()
        r = _step(cfg, ex, x, M, k, mode=mode, keep=("token_out",))
        outs[mode] = (x.cpu().numpy(), r)
    ws = {m: r["workspace_bytes"] for m, (_, r) in outs.items()}
    assert ws["fused"] < ws["mask_only"] < ws["eager"]
    xf, xm, xe = (outs[m][0] for m in ("fused", "mask_only", "eager"))
    # same number committed; positions agree up to bf16-logits near-ties
    for xo in (xf, xm, xe):
        assert (xo == MASK_ID).sum() == M - k
    agree = ((xf != MASK_ID) & (xm != MASK_ID)).sum()
    assert agree >= k - 3
    both = (xf != MASK_ID) & (xm != MASK_ID) & (x0.cpu().numpy() == MASK_ID)
    assert (xf[both] == xm[both]).mean() > 0.95


def test_denoising_run_unmasks_everything(env):
    """simulate_run with the execute hook: the whole linear schedule runs in the
    arena and every masked token is committed by the last step."""
    from paper_2601_06562_b200 import workload

    cfg, model, ex, dev = env
    scen = workload.ScenarioConfig(2048, 0.5, 8, budget=model.nbytes() + (32 << 20))
    x = _x(2048, scen.output_length, dev, seed=5)
    seen = []

    def execute(step, g, table, plan, config):
        k = scen.unmask_count(step)
        before = int((x == MASK_ID).sum())
        r = ex.run(g, x, k, table=table, plan=plan)
        after = int((x == MASK_ID).sum())
        assert before == g.bindings["M"] and before - after == k
        seen.append((config.k_logits, config.k_ffn))
        return {"ms": r["ms"], "committed": r["committed_bytes"]}

    res = workload.simulate_run(cfg, scen, execute=execute)
    assert int((x == MASK_ID).sum()) == 0
    assert all(r.measured["committed"] >= r.metrics.theoretical_peak for r in res)
    assert len(seen) == 8


@pytest.mark.parametrize("K", [(1, 1), (3, 2)])
def test_fused_gather_template_matches_fused(env, K):
    """logits_mode='fused_gather' (K3 reads h at mask_idx; no hc tensor in the
    plan) commits exactly what the buffered fused template commits."""
    cfg, model, ex, dev = env
    L, M, k = 2048, 1024, 64
    x0 = _x(L, M, dev, seed=9)
    res = {}
    for mode in ("fused", "fused_gather"):
        x = x0.clone()
        r = _step(cfg, ex, x, M, k, K=K, mode=mode, keep=("token_out",))
        res[mode] = (x.cpu(), r["kept"]["token_out"].cpu(), r["kept"]["confidence"].cpu(), r["workspace_bytes"])
    for a, b in zip(res["fused"][:3], res["fused_gather"][:3]):
        assert torch.equal(a, b)
    assert res["fused_gather"][3] <= res["fused"][3]


def test_fused_ffn_forward_matches_plain_torch(native_lib):
    """fused_ffn=True: K10 gate/up GEMM with the SwiGLU epilogue inside the
    arena, against the plain-PyTorch forward of the same weights."""
    from paper_2601_06562_b200 import vmm, workload
    from paper_2601_06562_b200.executor import RandomDLLM, StepExecutor
    from torch_reference import reference_forward

    cfg = replace(workload.toy_configs()["tiny_llada"], fused_ffn=True)
    dev = torch.device("cuda", 0)
    model = RandomDLLM(cfg, dev, seed=4)
    ws = vmm.reserve(4 << 30, backend="cuda")
    try:
        ex = StepExecutor(model, ws, MASK_ID)
        L, M = 2048, 1024
        x = _x(L, M, dev, seed=3)
        ref = reference_forward(model, x.clone())
        for K in ((1, 1), (1, 3)):
            out = _step(cfg, ex, x.clone(), M, 16, K=K, keep=("l1.h_out",))
            torch.testing.assert_close(out["kept"]["l1.h_out"].float(), ref.float(), rtol=2e-2, atol=2e-2)
    finally:
        ws.close()
