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
    # one arena: the torch-scratch region, then the plan, committed to the granule
    assert out["committed_bytes"] >= out["scratch_bytes"] + out["workspace_bytes"]
    assert out["committed_bytes"] - out["scratch_bytes"] - out["workspace_bytes"] < ex.ws.page_size


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
    # selection vs the fp64 rule (positions make the rows differ, so the check is
    # not vacuous): equal outside the near-tie band of twice the measured error
    # (>= 1e-6), which holds few rows; swaps inside it are fp32 accumulation order
    err = float(np.max(np.abs(conf - ref["conf"]) / ref["conf"]))
    par = orc.selection_parity(sel_dev, conf, ref["conf"], ref["idx"], k, max(1e-6, 2 * err))
    assert err < 1e-4 and par["outside_band_equal"], par
    assert par["mismatches"] <= par["band_rows"] < 0.05 * M, par


def test_modes_agree(env):
    """fused (K2-K5) vs the reference's materialising mask-only and eager modes,
    each against the fp64 oracle on the same final hidden states. The fused
    mode holds fp32 statistics: its selection equals the fp64 rule outside a
    band of twice its measured error (>= 1e-6), holding few rows. The materialising modes round the logits to bf16 (the `logits`
    tensor's element_size 2, mosaic/workload.py:276) before the fp32 softmax,
    so their confidences carry that rounding: each mode's selection must equal
    the fp64 rule outside a band of twice its own measured confidence error,
    and its tokens must be exact where the fp64 margin exceeds the bf16
    rounding of two logits (1e-2 at these logit magnitudes)."""
    cfg, model, ex, dev = env
    L, M, k = 2048, 1024, 32
    x0 = _x(L, M, dev, seed=2)
    x0n = x0.cpu().numpy()
    idx = orc.mask_compact(x0n, MASK_ID)
    outs = {}
    for mode in ("fused", "mask_only", "eager"):
        x = x0.clone()
        r = _step(cfg, ex, x, M, k, mode=mode, keep=("token_out", "l1.h_out"))
        outs[mode] = (x.cpu().numpy(), r)
    ws = {m: r["workspace_bytes"] for m, (_, r) in outs.items()}
    assert ws["fused"] < ws["mask_only"] < ws["eager"]
    h = outs["fused"][1]["kept"]["l1.h_out"]
    for mode in ("mask_only", "eager"):  # the forward is the same in every mode
        assert torch.equal(outs[mode][1]["kept"]["l1.h_out"], h)
    ref = orc.softmax_stats(orc.logits_f64(h.float().cpu().numpy()[idx], model.w_vocab.float().cpu().numpy()))
    for mode, (xo, r) in outs.items():
        tok = r["kept"]["token_out"].cpu().numpy()
        conf = r["kept"]["confidence"].cpu().numpy()
        if mode == "eager":  # per-position rows: the masked ones
            tok, conf = tok[idx], conf[idx]
        sel = xo[idx] != MASK_ID
        assert (xo == MASK_ID).sum() == M - k and sel.sum() == k
        err = float(np.max(np.abs(conf - ref["conf"]) / ref["conf"]))
        par = orc.selection_parity(sel, conf, ref["conf"], idx, k, max(1e-6, 2 * err))
        assert par["outside_band_equal"], (mode, par)
        if mode == "fused":
            assert err < 1e-4 and par["band_rows"] < 0.05 * M, par
        margin = 1e-3 if mode == "fused" else 1e-2
        ok = ref["margin"] > margin
        assert np.array_equal(tok[ok], ref["arg"][ok]), mode


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


@pytest.mark.parametrize("name", ["tiny_2k", "llada_32k_1layer"])
def test_step_runs_in_one_arena(native_lib, name):
    """north_star (3) / mosaic/vmm.py:48-147: the whole step runs out of the one
    preplanned cuMem arena. Activations sit at their first-fit offsets; the
    torch-side temporaries of library calls (attention outputs) are carved from
    the arena's scratch region through csrc/pool.cu. After the first step,
    steps 2..N make no allocator calls at all: torch's segment and reserved-byte
    counters, the pool's allocation count and the arena's commitment stay
    fixed, and the pool never refused a request."""
    from paper_2601_06562_b200 import vmm, workload
    from paper_2601_06562_b200.executor import RandomDLLM, StepExecutor

    dev = torch.device("cuda", 0)
    if name == "tiny_2k":  # configs[0]
        cfg, L, layers, mask_id = replace(workload.toy_configs()["tiny_llada"], fused_ffn=True), 2048, None, MASK_ID
    else:  # configs[1]: LLaDA-8B widths and head at 32k, one layer executed (memory per layer is identical)
        cfg = workload.ModelConfig("llada_8b", 32, 4096, 12288, 32, 126464, 2, 0, True, "fused", "none",
                                   fused_ffn=True)
        L, layers, mask_id = 32768, 1, 126336
    model = RandomDLLM(cfg, dev, seed=1, distinct_layers=1)
    ws = vmm.reserve(24 << 30, backend="cuda")
    try:
        ex = StepExecutor(model, ws, mask_id, exec_layers=layers)
        M = L // 2
        g = workload.build_layer_template(cfg).instantiate({"L": L, "M": M, "K_logits": 1, "K_FFN": 2})
        table, plan = ex.plan(g)
        x0 = torch.randint(0, mask_id, (L,), dtype=torch.int32, device=dev)
        x0[L - M:] = mask_id
        x = torch.empty_like(x0)
        snaps = []
        for _ in range(4):
            x.copy_(x0)
            r = ex.run(g, x, 8, table=table, plan=plan)
            torch.cuda.synchronize()
            st = torch.cuda.memory_stats(dev)
            snaps.append((st["segment.all.current"], st["reserved_bytes.all.current"], st["num_alloc_retries"],
                          r["pool"]["allocs"], r["committed_bytes"]))
            assert r["pool"]["refused"] == 0
            assert r["committed_bytes"] == r["scratch_bytes"] + -(-plan.workspace_size // ws.page_size) * ws.page_size
            assert r["pool"]["high_water"] <= r["scratch_bytes"]
        assert len(set(snaps[1:])) == 1, snaps
        assert snaps[0][3] >= 1  # the attention temporaries really went through the arena's pool
    finally:
        ws.close()
