"""Maximum context length on one B200: the planned pipeline vs the eager
dense-logits baseline (BASELINE.json configs[4], north_star "15x longer
context" claim).

    python bench_context.py [--lengths 32768,262144,...] [--exec-layers 1] [--out FILE]

Pipeline arm: LLaDA-8B shape (32 layers, d 4096, d_ff 12288, V 126464), all
32 layers of random-init bf16 weights resident. Per length L (r_p = 0.5, so
M = L/2 at step 0): the lazy chunk search picks (K_logits, K_FFN) under the
device budget (free HBM after weights minus a fixed reserve for the CUDA
context, cuBLAS and attention temporaries), the first-fit plan is committed in
the cuMem arena, and one full step runs through the executor: forward of the
first ``--exec-layers`` layers (attention cost is quadratic, so deeper stacks
at millions of tokens take hours; the planned peak is per-layer identical, so
the memory footprint does not depend on the executed depth), chunked FFN, and
the fused K1-K5 logits + remask path.

Baseline arm: the same model in eager PyTorch (caching allocator, no plan, no
chunking): full [L, V] bf16 logits for every position, an fp32 softmax over
them (the usual sampler), confidence/argmax, then the remask. Its L_max is
found by bisection on torch.cuda.OutOfMemoryError.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import torch
import torch.nn.functional as F

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MASK_ID = 126336
RESERVE = 4 << 30  # CUDA context, cuBLAS workspace, side buffers (attention temporaries: the arena's scratch)


def llada_cfg(weights_bytes: int):
    from paper_2601_06562_b200 import workload

    return workload.ModelConfig("llada_8b", 32, 4096, 12288, 32, 126464, 2, weights_bytes, True, "fused", "none",
                                fused_ffn=True)


def make_x(L: int, M: int, dev) -> torch.Tensor:
    x = torch.randint(0, 126000, (L,), dtype=torch.int32, device=dev)
    x[L - M:] = MASK_ID
    return x


def pipeline_probe(ex, cfg, L: int, act_budget: int) -> dict:
    from paper_2601_06562_b200 import chunker, workload

    M = round(0.5 * L)
    tmpl = workload.build_layer_template(cfg)
    t0 = time.time()
    scratch = ex.scratch_bytes_for(L)  # the arena's torch-scratch region comes out of the same budget
    out = chunker.search_bottleneck(tmpl, {"L": L, "M": M}, act_budget - scratch)
    plan_s = time.time() - t0
    rec = {"L": L, "M": M, "feasible_plan": out.feasible, "reason": out.reason, "planned_peak": out.final_peak,
           "floor": out.floor, "plan_seconds": plan_s}
    if not out.feasible:
        return rec
    g = tmpl.instantiate({"L": L, "M": M, "K_logits": out.config.k_logits, "K_FFN": out.config.k_ffn})
    table, plan = ex.plan(g)
    x = make_x(L, M, ex.device)
    torch.cuda.reset_peak_memory_stats()
    base_res = torch.cuda.memory_reserved()
    k = max(1, M // 64)
    try:
        r = ex.run(g, x, k, table=table, plan=plan)
        ok = int((x == MASK_ID).sum()) == M - k
        # torch-side temporaries are served from the arena's scratch region (MemPool): only
        # growth of torch's reserve beyond those segments lies outside the arena
        outside = max(0, torch.cuda.max_memory_reserved() - base_res - r["pool"]["in_use"])
        rec.update({"ran": True, "ok": ok, "ms": r["ms"], "k": [out.config.k_logits, out.config.k_ffn],
                    "workspace_bytes": plan.workspace_size, "committed_bytes": r["committed_bytes"],
                    "scratch_region_bytes": r["scratch_bytes"], "scratch_high_water": r["pool"]["high_water"],
                    "outside_arena_bytes": outside,
                    "activation_gb": (r["committed_bytes"] + outside) / 1e9})
    except torch.cuda.OutOfMemoryError as exc:
        rec.update({"ran": False, "ok": False, "error": str(exc).splitlines()[0]})
    del x
    torch.cuda.empty_cache()
    return rec


def eager_step(model, x: torch.Tensor, M: int, exec_layers: int) -> None:
    """Plain PyTorch dLLM step with dense logits (the unchunked baseline)."""
    cfg = model.cfg
    L, d, H = x.numel(), cfg.d_model, cfg.n_heads
    h = model.w_embed.index_select(0, x)
    for i in range(exec_layers):
        lw = model.layer(i)
        q, kk, v = (h @ lw["w_qkv"][:, j * d:(j + 1) * d] for j in range(3))
        qh, kh, vh = (t.view(L, H, d // H).transpose(0, 1).unsqueeze(0) for t in (q, kk, v))
        a = F.scaled_dot_product_attention(qh, kh, vh).squeeze(0).transpose(0, 1).reshape(L, d)
        del q, kk, v, qh, kh, vh
        h = h + a @ lw["w_attn_out"]
        del a
        f = cfg.d_ff  # the same weights, from the K10 layouts (gate/up interleaved in 128-row blocks, down K-major)
        gu = lw["w_gate_up"].view(f // 128, 2, 128, d)
        act = F.silu(h @ gu[:, 0].reshape(f, d).t()) * (h @ gu[:, 1].reshape(f, d).t())
        h = h + act @ lw["w_down"].t()
        del act
    logits = h @ model.w_vocab.t()                      # [L, V] bf16, every position
    probs = torch.softmax(logits.float(), dim=-1)      # fp32 sampler
    conf, tok = probs.max(dim=-1)
    del probs, logits
    masked = (x == MASK_ID).nonzero().squeeze(1)
    kk = max(1, M // 64)
    sel = masked[torch.topk(conf[masked], kk).indices]
    x[sel] = tok[sel].to(torch.int32)


def baseline_probe(model, L: int, exec_layers: int) -> bool:
    M = round(0.5 * L)
    try:
        x = make_x(L, M, model.w_embed.device)
        eager_step(model, x, M, exec_layers)
        torch.cuda.synchronize()
        ok = True
    except torch.cuda.OutOfMemoryError:
        ok = False
    torch.cuda.empty_cache()
    return ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lengths", default="32768,262144,1048576")
    ap.add_argument("--exec-layers", type=int, default=1)
    ap.add_argument("--no-lmax-run", action="store_true")
    ap.add_argument("--out", default="gpurun_out/context_sweep.json")
    args = ap.parse_args()

    from paper_2601_06562_b200 import _build, vmm, workload
    from paper_2601_06562_b200.executor import RandomDLLM, StepExecutor

    _build.build()
    code_hash = _build.source_hash()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    total = torch.cuda.get_device_properties(dev).total_memory
    cfg0 = llada_cfg(0)
    model = RandomDLLM(cfg0, dev, seed=0)  # all 32 layers resident
    torch.cuda.synchronize()
    wbytes = model.nbytes()
    cfg = llada_cfg(wbytes)
    free, _ = torch.cuda.mem_get_info()
    act_budget = free - RESERVE
    ws = vmm.reserve(act_budget + (1 << 30), backend="cuda")
    ex = StepExecutor(model, ws, MASK_ID, exec_layers=args.exec_layers)
    # the arena holds the plan AND the torch-scratch region (attention temporaries): the
    # planner's budget is what is left after the region a step at L >= 32k starts with
    scratch = ex.scratch_bytes_for(1 << 22)
    plan_budget = act_budget - scratch
    result = {"device_total_bytes": total, "weights_bytes": wbytes, "free_after_weights": free,
              "reserve_bytes": RESERVE, "activation_budget": act_budget, "scratch_region_first_step": scratch,
              "exec_layers": args.exec_layers, "model": cfg.to_json_dict(), "code_hash": code_hash}
    t0 = time.time()
    result["planned_lmax"] = {
        "fused_chunking": workload.find_lmax(cfg, 0.5, plan_budget + wbytes, logits_mode="fused",
                                             peaks_monotone=False),
        "fused_no_chunking": workload.find_lmax(cfg, 0.5, plan_budget + wbytes, ("global_plan", "mask_only"),
                                                logits_mode="fused", peaks_monotone=False),
        "mask_only_chunking": workload.find_lmax(cfg, 0.5, plan_budget + wbytes, logits_mode="mask_only",
                                                 peaks_monotone=False),
        "eager_global_plan": workload.find_lmax(cfg, 0.5, plan_budget + wbytes, ("global_plan",),
                                                peaks_monotone=False),
        "seconds": time.time() - t0,
    }
    print(json.dumps(result["planned_lmax"]), flush=True)

    lengths = [int(s) for s in args.lengths.split(",") if s]
    lmax = result["planned_lmax"]["fused_chunking"]
    if not args.no_lmax_run:
        lengths.append(lmax)
    runs = []
    for L in lengths:
        rec = pipeline_probe(ex, cfg, L, act_budget)
        runs.append(rec)
        print(json.dumps(rec), flush=True)
    over = pipeline_probe(ex, cfg, int(lmax * 1.02) + 1, act_budget)  # just past the plan's limit
    result["pipeline"] = runs
    result["pipeline_past_lmax"] = over
    ws.close()  # the executor's scratch pool lets go of the arena first (Workspace.on_close)
    torch.cuda.empty_cache()

    # baseline: bisection on OOM
    lo, hi = 16384, 16384
    while baseline_probe(model, hi, args.exec_layers):
        lo, hi = hi, hi * 2
        if hi > (1 << 22):
            break
    while hi - lo > 4096:
        mid = (lo + hi) // 2
        lo, hi = (mid, hi) if baseline_probe(model, mid, args.exec_layers) else (lo, mid)
    result["baseline_lmax"] = lo
    measured = max((r["L"] for r in runs if r.get("ok")), default=0)
    result["pipeline_lmax_measured"] = measured
    result["ratio_measured"] = measured / lo if lo else None
    print(json.dumps({"baseline_lmax": lo, "pipeline_lmax_measured": measured,
                      "ratio": result["ratio_measured"]}), flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(result, indent=1) + "\n")


if __name__ == "__main__":
    main()
