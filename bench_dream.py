"""Dream-7B step at 128k tokens on one B200 (BASELINE.json configs[2]): the
lazily chunked FFN / logits inside the preplanned cuMem arena, Dream's
token-level shift as a row remap, and the vocab-sharded LM head measured per
rank shard.

    python bench_dream.py [--seq 131072] [--layers 28] [--out FILE]

Model: Dream-7B shape (28 layers, d 3584, d_ff 18944, 28 heads, V 152064;
BASELINE's vocab), random-init bf16 weights, ``shift_mode="in_place"`` (the
masked position p reads hidden row max(p-1, 0)), ``fused_ffn=True`` (K10
gate/up GEMM with the SwiGLU epilogue; K10 down GEMM with the residual
epilogue, which also does the chunk write and the residual add). One denoising step at
L = seq, r_p = 0.5 (M = L/2), k = M/64, run twice through the executor:

* ``unchunked``: K = (1, 1);
* ``searched``: the reference's lazy bottleneck search under an activation
  budget halfway between the non-chunkable floor and the unchunked peak
  (so the search must chunk).

Vocab sharding at P = 2/4/8 needs P GPUs; on one GPU this script measures
what each rank's device would run -- K3 + K4 over its V/P shard for the
step's M rows, plus the replicated K1/K2/K5 -- and reports the per-rank
hot-path time next to the 1-GPU one (the exchange itself, 12 B per row per
rank over NVLink, is not measured here; ``bench.py --gpus P`` under torchrun
measures the whole thing).
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MASK_ID = 151666


def dream_cfg(layers: int):
    from paper_2601_06562_b200 import workload

    return workload.ModelConfig("dream_7b", layers, 3584, 18944, 28, 152064, 2, 0, True, "fused", "in_place",
                                fused_ffn=True)


def run(ex, tmpl, L, M, K, profile=True):
    g = tmpl.instantiate({"L": L, "M": M, "K_logits": K[0], "K_FFN": K[1]})
    table, plan = ex.plan(g)
    k = max(1, M // 64)
    x = torch.randint(0, 151000, (L,), dtype=torch.int32, device=ex.device)
    x[L - M:] = MASK_ID
    ex.run(g, x.clone(), k, table=table, plan=plan)  # warm-up (cuBLAS / SDPA autotune, arena commit)
    xx = x.clone()
    r = ex.run(g, xx, k, table=table, plan=plan, profile=profile)
    assert int((xx == MASK_ID).sum()) == M - k
    hot = sum(r["ms_by_kind"].get(kd, 0.0) for kd in ("gather", "lmhead_stats", "sample", "commit"))
    ffn = sum(r["ms_by_kind"].get(kd, 0.0) for kd in ("ffn_gate_up", "ffn_up", "ffn_gate", "glu", "ffn_down",
                                                       "ffn_down_res", "chunk_write", "identity"))
    return {"K": list(K), "step_ms": r["ms"], "workspace_bytes": plan.workspace_size,
            "committed_bytes": r["committed_bytes"], "hot_path_ms": hot, "ffn_ms": ffn,
            "ms_by_kind": {kk: round(v, 3) for kk, v in r["ms_by_kind"].items()}}


def shard_times(M, d, V, dev):
    """Per-rank K3+K4 at V/P (P = 1, 2, 4, 8) for M rows, CUDA events."""
    from paper_2601_06562_b200 import hotpath

    g = torch.Generator(device=dev).manual_seed(3)
    hc = torch.randn(M, d, generator=g, device=dev).to(torch.bfloat16)
    W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
    out = {}
    for P in (1, 2, 4, 8):
        v = V // P
        Ws = W[:v]
        S, _ = hotpath.lmhead_plan(M, v, d)
        pm = torch.empty(S, M, device=dev)
        ps = torch.empty(S, M, device=dev)
        pa = torch.empty(S, M, device=dev, dtype=torch.int32)
        tok = torch.empty(M, dtype=torch.int32, device=dev)
        lse = torch.empty(M, device=dev)
        conf = torch.empty(M, device=dev)
        # the schedule MaskOnlyHead would pick for this rank's shard
        die = hotpath.die_map(dev)[0] if hotpath.die_aware_default(None, M, v) else None
        sched = torch.zeros(4, dtype=torch.int32, device=dev)

        def step():
            hotpath.lmhead_stats(hc, Ws, S, pm, ps, pa, m_host=M, die_of_sm=die, sched=sched)
            hotpath.stats_merge(pm, ps, pa, S, M, M, m_host=M, token=tok, lse=lse, conf=conf)

        for _ in range(2):
            step()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            step()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        out[f"P{P}"] = {"vocab_shard": v, "k3_k4_ms": ms, "tflops": 2.0 * M * d * v / ms / 1e9,
                        "k3_schedule": "dynamic die-aware" if die is not None else "dynamic"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=131072)
    ap.add_argument("--layers", type=int, default=28)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    from paper_2601_06562_b200 import _build, chunker, vmm, workload
    from paper_2601_06562_b200.executor import RandomDLLM, StepExecutor

    _build.build()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = dream_cfg(args.layers)
    model = RandomDLLM(cfg, dev, seed=5)
    weights_bytes = model.nbytes()
    tmpl = workload.build_layer_template(cfg)
    L, M = args.seq, round(0.5 * args.seq)
    ws = vmm.reserve(120 << 30, backend="cuda")
    ex = StepExecutor(model, ws, MASK_ID)
    full = run(ex, tmpl, L, M, (1, 1))
    peak = chunker.evaluate_peak(tmpl, {"L": L, "M": M}, chunker.ChunkConfig(1, 1))
    budget = (peak.total_peak + peak.non_chunkable_peak) // 2
    srch = chunker.search_bottleneck(tmpl, {"L": L, "M": M}, budget)
    ws.close()
    ws = vmm.reserve(120 << 30, backend="cuda")
    ex = StepExecutor(model, ws, MASK_ID)
    searched = run(ex, tmpl, L, M, (srch.config.k_logits, srch.config.k_ffn))
    ws.close()
    del ex, model
    torch.cuda.empty_cache()
    shards = shard_times(M, cfg.d_model, cfg.vocab_size, dev)
    replicated = full["hot_path_ms"] - full["ms_by_kind"].get("lmhead_stats", 0.0) - full["ms_by_kind"].get("sample", 0.0)
    line = {
        "workload": "dream7b_128k_mask50_shift",
        "config": {"n_layers": cfg.n_layers, "d_model": cfg.d_model, "d_ff": cfg.d_ff, "vocab": cfg.vocab_size,
                   "seq_len": L, "masked": M, "unmask_k": max(1, M // 64), "shift_mode": cfg.shift_mode},
        "data": "synthetic (random-init bf16 weights, random tokens; no checkpoint)",
        "weights_bytes": weights_bytes,
        "unchunked": full,
        "searched": {**searched, "budget_bytes": budget, "search_reason": srch.reason,
                     "evaluations": srch.evaluations, "planned_peak": srch.final_peak},
        "chunking_overhead": searched["step_ms"] / full["step_ms"] - 1.0,
        "activation_saving": 1.0 - searched["workspace_bytes"] / full["workspace_bytes"],
        "vocab_sharded_per_rank": shards,
        "replicated_hot_path_ms": replicated,
        "note": "per-rank K3+K4 measured on one GPU at the rank's vocab shard; the all-gather of 12 B/row/rank "
                "triples is not included (needs P GPUs)",
    }
    print(json.dumps(line), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(line, indent=1))


if __name__ == "__main__":
    main()
