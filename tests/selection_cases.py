"""Remask-selection parity cases at BASELINE.json configs (test
infrastructure, shared by tests/test_gpu_selection.py and
scripts/selection_parity.py, which writes the profiles/ record).

Each case runs the fused step on the B200, then recomputes the fp64
confidences of EVERY masked row on the host with the CPU oracle
(``softmax_stats_blocked``: fp64 BLAS over the same bf16 operands) and
compares the device's committed set with the fp64 rule's
(``selection_parity``: exact mismatch count, rows inside the near-tie band).

Configs (BASELINE.json):
* configs[0] ``tiny``: the 2-layer d-256 model's random-init forward in the
  cuMem arena (with rotary positions, so masked rows differ), L 2048, M 1024;
* configs[1] ``llada_32k``: LLaDA-8B head (d 4096, V 126464), L 32768, M 16384;
* configs[2] ``dream_128k``: Dream-7B head (d 3584, V 152064, token shift),
  L 131072, M 65536.
Unmask counts follow the reference schedule (mosaic/workload.py:140-146) with
64 steps, step 0: 256 (LLaDA), 1024 (Dream); 64 at the tiny config (16 steps).
"""
from __future__ import annotations

import time

import numpy as np
import torch

import mosaic_oracle as orc

BAND_REL = 1e-6  # near-tie band around the k-th fp64 confidence
CONF_REL = 1e-4  # measured confidence error bound: 5.6e-7 at d 256, 3.0-3.4e-5 at d 3584/4096 (tensor-core
# fp32 accumulation over K = d; the north_star tolerance is 1e-3)

HEADS = {
    "llada_32k": dict(L=32768, d=4096, V=126464, shift=False, k=orc.unmask_counts(32768, 0.5, 64)[0]),
    "dream_128k": dict(L=131072, d=3584, V=152064, shift=True, k=orc.unmask_counts(131072, 0.5, 64)[0]),
}


def _mask(x: torch.Tensor, M: int, layout: str, g: torch.Generator, mask_id: int) -> None:
    L = x.numel()
    if layout == "scattered":
        x[torch.randperm(L, generator=g, device=x.device)[:M]] = mask_id
    elif layout == "suffix":  # the step-0 layout of the reference schedule (prompt, then the masked answer)
        x[L - M:] = mask_id
    else:
        raise ValueError(layout)


def head_case(dev, name: str, layout: str, seed: int = 0) -> dict:
    """One fused step (K1-K5) at configs[1]/[2] size; every row against fp64."""
    from paper_2601_06562_b200 import MaskOnlyHead

    c = HEADS[name]
    L, d, V, shift, k = c["L"], c["d"], c["V"], c["shift"], c["k"]
    M = L // 2
    mask_id = V - 1
    g = torch.Generator(device=dev).manual_seed(1000 + seed + L)
    H = torch.randn(L, d, generator=g, device=dev).to(torch.bfloat16)
    W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
    x = torch.randint(0, V - 1, (L,), generator=g, device=dev, dtype=torch.int32)
    _mask(x, M, layout, g, mask_id)
    x0 = x.cpu().numpy()
    head = MaskOnlyHead(W, seq_len=L, mask_id=mask_id, shift=shift)
    out = head.step(x, H, k)
    torch.cuda.synchronize()
    Md = int(out.m_dev.item())
    idx = out.idx[:Md].cpu().numpy()
    dev_out = {n: getattr(out, n)[:Md].cpu().numpy() for n in ("token", "lse", "conf", "selected")}
    x1 = x.cpu().numpy()
    src = orc.source_rows(idx, shift)
    rows = H[torch.from_numpy(src).to(dev).long()].float().cpu().numpy()
    Wc = W.float().cpu().numpy()
    del head, H, W
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    ref = orc.softmax_stats_blocked(rows, Wc)
    oracle_s = time.perf_counter() - t0
    return _record(name, layout, L, x0, x1, idx, mask_id, k, dev_out, ref, oracle_s)


def tiny_case(dev, seed: int = 3) -> dict:
    """configs[0]: the tiny model's forward in the arena (StepExecutor), then
    the hot path on its final hidden states; the executor's committed sequence
    must equal the head's, and the head's selection is checked against fp64."""
    from paper_2601_06562_b200 import MaskOnlyHead, vmm, workload
    from paper_2601_06562_b200.executor import RandomDLLM, StepExecutor

    cfg = workload.toy_configs()["tiny_llada"]
    L, M, k, mask_id = 2048, 1024, 64, 8191
    model = RandomDLLM(cfg, dev, seed=seed)
    ws = vmm.reserve(1 << 30, backend="cuda")
    try:
        rng = np.random.default_rng(seed)
        x0 = rng.integers(0, mask_id, size=L).astype(np.int32)
        x0[L - M:] = mask_id
        g = workload.build_layer_template(cfg).instantiate({"L": L, "M": M, "K_logits": 1, "K_FFN": 1})
        xe = torch.from_numpy(x0).to(dev)
        r = StepExecutor(model, ws, mask_id).run(g, xe, k, keep=(f"l{cfg.n_layers - 1}.h_out",))
        h = r["kept"][f"l{cfg.n_layers - 1}.h_out"]
        head = MaskOnlyHead(model.w_vocab, seq_len=L, mask_id=mask_id)
        x = torch.from_numpy(x0).to(dev)
        out = head.step(x, h, k)
        torch.cuda.synchronize()
        Md = int(out.m_dev.item())
        idx = out.idx[:Md].cpu().numpy()
        dev_out = {n: getattr(out, n)[:Md].cpu().numpy() for n in ("token", "lse", "conf", "selected")}
        x1 = x.cpu().numpy()
        executor_equal = bool(np.array_equal(x1, xe.cpu().numpy()))
        rows = h.float().cpu().numpy()[idx]
        t0 = time.perf_counter()
        ref = orc.softmax_stats_blocked(rows, model.w_vocab.float().cpu().numpy())
        rec = _record("tiny", "suffix", L, x0, x1, idx, mask_id, k, dev_out, ref, time.perf_counter() - t0)
        rec["executor_commit_equals_head"] = executor_equal
        return rec
    finally:
        ws.close()


def _record(name, layout, L, x0, x1, idx, mask_id, k, dev_out, ref, oracle_s) -> dict:
    par = orc.selection_parity(dev_out["selected"], dev_out["conf"], ref["conf"], idx, k, BAND_REL)
    ok = ref["margin"] > 1e-3
    sel = dev_out["selected"].astype(bool)
    # the committed tokens are the device argmax of exactly the selected rows
    commit_ok = bool(np.array_equal(x1[idx[sel]], dev_out["token"][sel]) and np.all(x1[idx[~sel]] == mask_id)
                     and np.array_equal(np.delete(x1, idx), np.delete(x0, idx)))
    err = par["conf_max_rel_err"]
    m_dev = dev_out["lse"].astype(np.float64) + np.log(dev_out["conf"].astype(np.float64))  # max logit = lse + ln p
    return {
        "config": name, "layout": layout, "L": int(L), **par,
        # rows an error of twice the measured one could reorder around the k-th fp64 confidence
        "band_rows_at_2x_conf_err": int(orc.near_tie_rows(ref["conf"], k, 2 * err).sum()),
        "max_logit_abs_err": float(np.max(np.abs(m_dev - ref["max"]))),
        "lse_abs_err": float(np.max(np.abs(dev_out["lse"] - ref["lse"]))),
        "indices_equal": bool(np.array_equal(idx, orc.mask_compact(x0, mask_id))),
        "tokens_equal_where_margin_gt_1e-3": bool(np.array_equal(dev_out["token"][ok], ref["arg"][ok])),
        "rows_margin_gt_1e-3": int(ok.sum()),
        "token_mismatch_rows_margin_le_1e-3": int((dev_out["token"][~ok] != ref["arg"][~ok]).sum()),
        "lse_max_rel_err": float(np.max(np.abs(dev_out["lse"] - ref["lse"]) / np.abs(ref["lse"]))),
        "commit_consistent": commit_ok,
        "oracle": "fp64 BLAS over the bf16 operands, every masked row (oracle.softmax_stats_blocked)",
        "oracle_s": round(oracle_s, 2),
    }


def check(rec: dict) -> None:
    """The parity bar (north_star): indices bit-exact; the committed set equal
    to the fp64 rule's (zero mismatches; a fortiori outside the 1e-6 band);
    tokens exact where the margin > 1e-3; lse and confidence well inside the
    1e-3 relative tolerance."""
    assert rec["indices_equal"], rec
    assert rec["commit_consistent"], rec
    assert rec["conf_max_rel_err"] < CONF_REL, rec
    assert rec["outside_band_equal"], rec
    assert rec["mismatches"] == 0, rec
    assert rec["tokens_equal_where_margin_gt_1e-3"], rec
    assert rec["lse_max_rel_err"] < 1e-3, rec
