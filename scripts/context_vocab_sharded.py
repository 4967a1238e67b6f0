"""Planned maximum context per rank of a vocab-sharded LLaDA-8B run (BASELINE.json
configs[4] "on 1 and 8 B200"), from a bench_context.py sweep record.

Vocab sharding (north_star item 4) splits only the LM head: every rank keeps
the full forward, the FFN chunks and the [M, 3S] partials, so its activation
plan is the 1-GPU plan and its budget grows only by the (P-1)/P of the LM head
it no longer holds. The per-rank L_max is therefore the planner's answer
(workload.find_lmax, the same call bench_context.py measures at P = 1) under
that budget -- a planned figure, since no multi-GPU box was available.

    python scripts/context_vocab_sharded.py profiles/r02c_context_sweep.json
"""
from __future__ import annotations

import json
import sys
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(path: str) -> None:
    from paper_2601_06562_b200 import workload

    rec = json.loads(Path(path).read_text())
    m = rec["model"]
    cfg = workload.ModelConfig(m["name"], m["n_layers"], m["d_model"], m["d_ff"], m["n_heads"], m["vocab_size"],
                               m["element_size"], m["weights_bytes"], m["gated_ffn"], m["logits_mode"],
                               m["shift_mode"], fused_splits=m["fused_splits"], fused_ffn=m["fused_ffn"])
    head = cfg.vocab_size * cfg.d_model * cfg.element_size
    plan_budget = rec["activation_budget"] - rec["scratch_region_first_step"]
    out = {}
    for P in (1, 2, 4, 8):
        freed = head - head // P
        w = cfg.weights_bytes - freed
        lmax = workload.find_lmax(replace(cfg, weights_bytes=w), 0.5, plan_budget + freed + w,
                                  logits_mode="fused", peaks_monotone=False)
        out[str(P)] = {"weights_bytes_per_rank": w, "activation_budget_per_rank": plan_budget + freed,
                       "planned_lmax": lmax}
    rec["planned_lmax_vocab_sharded"] = {
        "per_rank": out,
        "note": "vocab sharding splits the LM head only; activations are replicated, so the per-rank L_max is the "
                "1-GPU plan under a budget larger by the LM-head bytes a rank no longer holds (planned, "
                "workload.find_lmax; no multi-GPU box)"}
    Path(path).write_text(json.dumps(rec, indent=1) + "\n")
    print(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1])
