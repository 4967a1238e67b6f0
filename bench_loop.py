"""The whole denoising loop on one B200: the reference's step loop
(`simulate_run`, mosaic/workload.py:349-399 -- per step: masked count -> lazy
chunk search -> instantiate -> liveness -> first-fit plan) with this
package's execute hook running every planned step on the device in the cuMem
arena until every masked position is committed.

    python bench_loop.py [--seq 32768] [--steps 64] [--layers 32] [--budget-gb G] [--out FILE]

Model: LLaDA-8B shape (32 layers, d 4096, d_ff 12288, V 126464; random-init
bf16; ``fused`` logits + ``fused_ffn``), r_p = 0.5 so the output half starts
masked and the linear schedule commits k_n tokens per step. Reports wall and
device time per step, the host planning time per step (search + instantiate
+ plan), the per-step chunk configs and committed arena bytes, and the
generation throughput (output tokens / total time). With ``--budget-gb`` the
search runs under that device budget (weights included), so later steps can
shrink their plans.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MASK_ID = 126336


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=32768)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--budget-gb", type=float, default=None)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    from paper_2601_06562_b200 import _build, vmm, workload
    from paper_2601_06562_b200.executor import RandomDLLM, StepExecutor

    _build.build()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg0 = workload.ModelConfig("llada_8b", args.layers, 4096, 12288, 32, 126464, 2, 0, True, "fused", "none",
                                fused_ffn=True)
    model = RandomDLLM(cfg0, dev, seed=2)
    wbytes = model.nbytes()
    cfg = workload.ModelConfig(**{**cfg0.__dict__, "weights_bytes": wbytes})
    budget = int(args.budget_gb * 1e9) if args.budget_gb else None
    scen = workload.ScenarioConfig(args.seq, 0.5, args.steps, budget=budget)
    x = torch.randint(0, 126000, (args.seq,), dtype=torch.int32, device=dev)
    x[args.seq - scen.output_length:] = MASK_ID
    free, _ = torch.cuda.mem_get_info()
    ws = vmm.reserve(free - (4 << 30), backend="cuda")
    ex = StepExecutor(model, ws, MASK_ID)

    # one untimed warm-up step (cuBLAS / SDPA autotune, arena first commit)
    g0 = workload.build_layer_template(cfg).instantiate({"L": args.seq, "M": scen.masked_at(0), "K_logits": 1,
                                                         "K_FFN": 1})
    ex.run(g0, x.clone(), 1)

    per_step = []
    t_plan = [time.perf_counter()]

    def execute(step, g, table, plan, config):
        t_exec = time.perf_counter()
        k = scen.unmask_count(step)
        before = int((x == MASK_ID).sum())
        r = ex.run(g, x, k, table=table, plan=plan)
        after = int((x == MASK_ID).sum())
        assert before - after == k, (step, before, after, k)
        per_step.append({"step": step, "M": g.bindings["M"], "k": k, "device_ms": r["ms"],
                         "plan_ms": (t_exec - t_plan[0]) * 1e3, "K": [config.k_logits, config.k_ffn],
                         "workspace_bytes": plan.workspace_size, "committed_bytes": r["committed_bytes"]})
        t_plan[0] = time.perf_counter()
        return {"ms": r["ms"]}

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    results = workload.simulate_run(cfg, scen, keep_traces=False, execute=execute)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    assert int((x == MASK_ID).sum()) == 0
    dev_ms = sum(s["device_ms"] for s in per_step)
    plan_ms = sum(s["plan_ms"] for s in per_step)
    line = {
        "workload": f"llada8b_{args.seq}_loop{args.steps}",
        "config": {"n_layers": args.layers, "seq_len": args.seq, "output_tokens": scen.output_length,
                   "steps": args.steps, "budget_bytes": budget, "logits_mode": "fused", "fused_ffn": True},
        "data": "synthetic (random-init bf16 weights, random prompt tokens; no checkpoint)",
        "weights_bytes": wbytes,
        "wall_s": wall, "device_s": dev_ms / 1e3, "planning_s": plan_ms / 1e3,
        "planning_share": plan_ms / (wall * 1e3),
        "output_tokens_per_s": scen.output_length / wall,
        "mean_par": sum(r.metrics.par for r in results) / len(results),
        "max_committed_bytes": max(s["committed_bytes"] for s in per_step),
        "steps_detail": per_step,
    }
    print(json.dumps({k: v for k, v in line.items() if k != "steps_detail"}), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(line, indent=1))
    ws.close()


if __name__ == "__main__":
    main()
