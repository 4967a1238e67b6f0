"""Serving-side benchmark beyond the reference's single sequence: semi-
autoregressive block decoding on the LLaDA-8B head (d 4096, V 126464).

For B sequences of Ls positions (the second half masked), one step decodes the
first `block` positions of every sequence's masked half:
  * batched   -- MaskOnlyHead.step_batch over all B blocks (one K1/K2/K3/K4 pass,
                 segmented K5: each sequence commits its own k), eager and as a
                 captured CUDA graph;
  * per-seq   -- B separate MaskOnlyHead.step(window=...) calls, each streaming the
                 whole 1.04 GB LM head for <= block rows.
Also one sampling (temperature 1) batched step. Synthetic bf16 hidden states and
a random-init head; CUDA events, median of repeated measurements.

    python bench_serving.py [--batches 1,8,32,64,128] [--block 32] [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def _time(fn, reps=5, iters=10):
    for _ in range(3):
        fn()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(iters):
            fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / iters)
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="1,8,32,64,128")
    ap.add_argument("--block", type=int, default=32)
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    from paper_2601_06562_b200 import MaskOnlyHead, _build

    _build.build()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    d, V, Ls, blk = 4096, 126464, args.seq, args.block
    mask_id = V - 1
    W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
    lo = Ls // 2
    one = MaskOnlyHead(W, seq_len=Ls, mask_id=mask_id)
    rows = []
    for B in (int(b) for b in args.batches.split(",") if b):
        H = torch.randn(B, Ls, d, generator=g, device=dev).to(torch.bfloat16)
        x0 = torch.randint(0, V - 1, (B, Ls), generator=g, device=dev, dtype=torch.int32)
        x0[:, lo:] = mask_id
        head = MaskOnlyHead(W, seq_len=B * blk, mask_id=mask_id)
        smp = MaskOnlyHead(W, seq_len=B * blk, mask_id=mask_id, temperature=1.0, seed=1)
        x = x0.clone()
        xg = x0.clone()
        graph = head.capture(xg, H, args.k, window=(lo, lo + blk))

        def batched():
            x.copy_(x0)
            head.step_batch(x, H, args.k, window=(lo, lo + blk))

        def batched_graph():
            xg.copy_(x0)
            graph.replay()

        def sampled():
            x.copy_(x0)
            smp.step_batch(x, H, args.k, window=(lo, lo + blk))

        def per_seq():
            x.copy_(x0)
            for b in range(B):
                one.step(x[b], H[b], args.k, window=(lo, lo + blk))

        t = {"batched_ms": _time(batched), "batched_graph_ms": _time(batched_graph),
             "batched_sampling_ms": _time(sampled), "per_sequence_ms": _time(per_seq, reps=3, iters=3)}
        t.update({"B": B, "block": blk, "masked_tokens_per_s": B * blk / (t["batched_ms"] / 1e3),
                  "speedup_vs_per_sequence": t["per_sequence_ms"] / t["batched_ms"]})
        rows.append(t)
        print(json.dumps(t), flush=True)
        del H, head, smp, graph
    if args.out:
        Path(args.out).write_text(json.dumps({"workload": "llada8b_head_block_decoding", "seq_len": Ls,
                                              "block": blk, "k": args.k,
                                              "data": "synthetic (random hidden states, random-init head)",
                                              "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
