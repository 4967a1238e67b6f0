"""Same-box A/B of K3's unit schedules -- static (pair c takes units c, c +
pairs, ...), dynamic (units claimed from a global counter), dynamic die-aware
(die-0 pairs claim from the front, die-1 pairs from the back) -- at the full and
per-rank vocab-shard shapes, alternating, CUDA events on the launching stream.

    python scripts/k3_die_ab.py [--reps 3]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--shapes", default="", help="comma-separated subset of the shape names")
    a = ap.parse_args()
    from paper_2601_06562_b200 import _build, hotpath

    _build.build()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    table, _ = hotpath.die_map(dev)
    sched = torch.zeros(4, dtype=torch.int32, device=dev)
    out = []
    shapes = (("llada_p1", 16384, 4096, 126464), ("llada_p8", 16384, 4096, 126464 // 8),
              ("dream_p1", 65536, 3584, 152064), ("dream_p2", 65536, 3584, 152064 // 2),
              ("dream_p4", 65536, 3584, 152064 // 4), ("dream_p8", 65536, 3584, 152064 // 8))
    only = set(a.shapes.split(",")) if a.shapes else None
    for name, M, d, V in shapes:
        if only and name not in only:
            continue
        hc = torch.randn(M, d, generator=g, device=dev).to(torch.bfloat16)
        W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
        S, _ = hotpath.lmhead_plan(M, V, d)
        pm, ps = torch.empty(S, M, device=dev), torch.empty(S, M, device=dev)
        pa = torch.empty(S, M, device=dev, dtype=torch.int32)
        res = {"static": [], "dynamic": [], "dynamic_die": []}
        for _ in range(a.reps):
            for mode in res:
                kw = ({} if mode == "static" else
                      dict(sched=sched) if mode == "dynamic" else dict(die_of_sm=table, sched=sched))
                for _ in range(3):
                    hotpath.lmhead_stats(hc, W, S, pm, ps, pa, m_host=M, **kw)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                s.record()
                for _ in range(a.iters):
                    hotpath.lmhead_stats(hc, W, S, pm, ps, pa, m_host=M, **kw)
                e.record()
                e.synchronize()
                ms = s.elapsed_time(e) / a.iters
                res[mode].append(round(2.0 * M * d * V / ms / 1e9, 1))
        rec = {"shape": name, "M": M, "d": d, "V": V, "splits": S, "tflops": res}
        print(json.dumps(rec), flush=True)
        out.append(rec)
        del hc, W


if __name__ == "__main__":
    main()
