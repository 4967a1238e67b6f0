"""LLaDA-MoE step on one B200 (BASELINE.json configs[3]): the chunked expert FFN
inside the preplanned cuMem arena, followed by the fused mask-only logits +
remask path.

    python bench_moe.py [--seq 65536] [--steps 2] [--warmup 1] [--out FILE]

Model: the reference's ``moe_like`` shape (configs/moe_like.json: 16 layers,
d 2048, d_ff 1408 per expert, 64 experts, top-8, 16 heads, V 126464), all
layer weights resident (random-init bf16). One denoising step at L = seq,
r_p = 0.5 (M = L/2 masked), k = M/64 tokens committed. Two plans are run:

* ``unchunked``: K = (1, 1) -- one FFN chunk of L*top_k dispatch rows;
* ``searched``: the reference's lazy bottleneck search (chunker.search_bottleneck)
  under an activation budget halfway between the non-chunkable floor and the
  unchunked peak, so the expert FFN must be chunked (K_FFN > 1).

The expert FFN runs as K10 grouped tcgen05 GEMMs over the K8 expert
segments (gate/up with the SwiGLU epilogue, then down), offsets on the device.

Each is timed on the device (CUDA events, max of ``--steps`` after
``--warmup``) with a per-op-kind breakdown; the JSON line reports the step
time, the chunk config, planned / committed arena bytes, the expert GEMM
TFLOP/s, K8/K9 bandwidth and the hot-path (K1-K5) share.
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MASK_ID = 126336


def moe_cfg():
    from paper_2601_06562_b200 import workload

    return workload.ModelConfig("llada_moe", 16, 2048, 1408, 16, 126464, 2, 0, True, "fused", "none",
                                workload.MoEConfig(64, 8))


def run_plan(ex, tmpl, L, M, K, steps, warmup):
    g = tmpl.instantiate({"L": L, "M": M, "K_logits": K[0], "K_FFN": K[1]})
    table, plan = ex.plan(g)
    k = max(1, M // 64)
    x0 = torch.randint(0, 126000, (L,), dtype=torch.int32, device=ex.device)
    x0[L - M:] = MASK_ID
    best = None
    for i in range(warmup + steps):
        x = x0.clone()
        r = ex.run(g, x, k, table=table, plan=plan, profile=(i >= warmup))
        assert int((x == MASK_ID).sum()) == M - k
        if i >= warmup and (best is None or r["ms"] < best["ms"]):
            best = r
    best["K"] = list(K)
    best["workspace_bytes"] = plan.workspace_size
    return best


def summarize(cfg, L, r):
    E, k = cfg.moe.n_experts, cfg.moe.top_k
    d, f, nl = cfg.d_model, cfg.d_ff, cfg.n_layers
    P = L * k
    byk = r["ms_by_kind"]
    gemm_ms = sum(byk.get(kd, 0.0) for kd in ("ffn_gate_up", "ffn_down"))  # K10 (gate/up + SwiGLU, down)
    gemm_flops = 3 * 2.0 * P * d * f * nl
    # K9 reads k rows of d + writes 1 row per token; K8 reads E fp32 logits per token
    k9_bytes = nl * L * (k + 1) * d * 2.0 + nl * L * k * 8.0
    k8_bytes = nl * L * (E * 4.0 + k * 16.0)
    hot = ("gather", "lmhead_stats", "sample", "commit")
    hot_ms = sum(byk.get(kd, 0.0) for kd in hot)
    return {
        "K": r["K"], "step_ms": r["ms"], "workspace_bytes": r["workspace_bytes"],
        "committed_bytes": r["committed_bytes"], "ms_by_kind": {kk: round(v, 3) for kk, v in byk.items()},
        "expert_gemm_ms": gemm_ms, "expert_gemm_tflops": gemm_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms else None,
        "k8_route_GBps": k8_bytes / (byk.get("moe_route", 0.0) / 1e3) / 1e9 if byk.get("moe_route") else None,
        "k9_combine_GBps": k9_bytes / (byk.get("moe_combine", 0.0) / 1e3) / 1e9 if byk.get("moe_combine") else None,
        "hot_path_ms": hot_ms,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=65536)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    from paper_2601_06562_b200 import _build, chunker, vmm, workload
    from paper_2601_06562_b200.executor import RandomDLLM, StepExecutor

    _build.build()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = moe_cfg()
    model = RandomDLLM(cfg, dev, seed=7)
    tmpl = workload.build_layer_template(cfg)
    L, M = args.seq, round(0.5 * args.seq)
    ws = vmm.reserve(96 << 30, backend="cuda")
    ex = StepExecutor(model, ws, MASK_ID)
    full = run_plan(ex, tmpl, L, M, (1, 1), args.steps, args.warmup)
    peak = chunker.evaluate_peak(tmpl, {"L": L, "M": M}, chunker.ChunkConfig(1, 1))
    budget = (peak.total_peak + peak.non_chunkable_peak) // 2
    out = chunker.search_bottleneck(tmpl, {"L": L, "M": M}, budget)
    ws.close()
    ws = vmm.reserve(96 << 30, backend="cuda")  # fresh arena: committed bytes of the searched plan alone
    ex = StepExecutor(model, ws, MASK_ID)
    searched = run_plan(ex, tmpl, L, M, (out.config.k_logits, out.config.k_ffn), args.steps, args.warmup)
    ws.close()
    a, b = summarize(cfg, L, full), summarize(cfg, L, searched)
    line = {
        "workload": "llada_moe_64k_mask50" if L == 65536 else f"llada_moe_{L}_mask50",
        "config": {"n_layers": cfg.n_layers, "d_model": cfg.d_model, "d_ff_expert": cfg.d_ff,
                   "n_experts": cfg.moe.n_experts, "top_k": cfg.moe.top_k, "vocab": cfg.vocab_size,
                   "seq_len": L, "masked": M, "unmask_k": max(1, M // 64)},
        "data": "synthetic (random-init bf16 weights, random tokens; no checkpoint)",
        "weights_bytes": model.nbytes(),
        "unchunked": a,
        "searched": {**b, "budget_bytes": budget, "search_reason": out.reason, "evaluations": out.evaluations,
                     "planned_peak": out.final_peak},
        "chunking_overhead": b["step_ms"] / a["step_ms"] - 1.0,
        "activation_saving": 1.0 - b["workspace_bytes"] / a["workspace_bytes"],
        "masked_tokens_per_s_step": M / (b["step_ms"] / 1e3),
    }
    print(json.dumps(line), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(line, indent=1))


if __name__ == "__main__":
    main()
