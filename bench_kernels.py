"""Per-kernel throughput at the BASELINE.json shapes (one B200), CUDA events on
the launching stream, inputs larger than L2 where the shape allows.

    python bench_kernels.py [--out gpurun_out/kernels.json]

K1/K2/K6 are reported as achieved HBM GB/s of algorithmic bytes against the
measured copy bandwidth; K3 as TFLOP/s against the measured bf16 peak; K4/K5
as latency.
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def timeit(fn, iters=20, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/kernels.json")
    args = ap.parse_args()
    from paper_2601_06562_b200 import _build, hotpath

    _build.build()
    dev = torch.device("cuda", 0)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    tf = peaks.get("bf16_tflops", 1590.0)
    out = {"peaks": {"hbm_gbs": hbm, "bf16_tflops": tf}}
    g = torch.Generator(device=dev).manual_seed(0)

    # K1 ---------------------------------------------------------------------
    for L in (32768, 1 << 20, 1 << 22):
        x = torch.randint(0, 1000, (L,), generator=g, device=dev, dtype=torch.int32)
        x[L // 2:] = 999999
        idx = torch.empty(L, dtype=torch.int32, device=dev)
        m = torch.zeros(1, dtype=torch.int32, device=dev)
        sc = torch.empty(hotpath.mask_compact_scratch_bytes(L), dtype=torch.uint8, device=dev)
        ms = timeit(lambda: hotpath.mask_compact(x, 999999, idx, m, sc))
        byts = 2 * 4 * L + 4 * (L // 2)  # x read twice + indices written
        out[f"k1_compact_L{L}"] = {"ms": ms, "GBps": byts / ms / 1e6, "frac_hbm": byts / ms / 1e6 / hbm}

    # K2 ---------------------------------------------------------------------
    for name, L, d in (("llada", 32768, 4096), ("dream", 131072, 3584)):
        M = L // 2
        H = torch.randn(L, d, generator=g, device=dev).to(torch.bfloat16)
        idx = torch.arange(L - M, L, device=dev, dtype=torch.int32)
        hc = torch.empty(M, d, device=dev, dtype=torch.bfloat16)
        ms = timeit(lambda: hotpath.gather_rows(H, idx, hc, m_host=M))
        byts = 2 * 2 * M * d + 4 * M
        out[f"k2_gather_{name}"] = {"ms": ms, "GBps": byts / ms / 1e6, "frac_hbm": byts / ms / 1e6 / hbm}
        del H, hc

    # K3 + K4 ----------------------------------------------------------------
    for name, M, d, V in (("llada", 16384, 4096, 126464), ("dream", 65536, 3584, 152064),
                          ("moe", 32768, 2048, 126464), ("tiny", 1024, 256, 8192),
                          ("llada_shard8", 16384, 4096, 126464 // 8)):
        hc = torch.randn(M, d, generator=g, device=dev).to(torch.bfloat16)
        W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
        S, tps = hotpath.lmhead_plan(M, V, d)
        pm = torch.empty(S, M, device=dev)
        ps = torch.empty(S, M, device=dev)
        pa = torch.empty(S, M, device=dev, dtype=torch.int32)
        it = 5 if M * V > 1e9 else 50
        die, sched = hotpath.die_map(dev)[0], torch.zeros(4, dtype=torch.int32, device=dev)
        # the product's dynamic unit schedule; the static one and the die-split dynamic one beside it
        ms = timeit(lambda: hotpath.lmhead_stats(hc, W, S, pm, ps, pa, m_host=M, sched=sched), iters=it)
        ms_static = timeit(lambda: hotpath.lmhead_stats(hc, W, S, pm, ps, pa, m_host=M), iters=it)
        ms_die = timeit(lambda: hotpath.lmhead_stats(hc, W, S, pm, ps, pa, m_host=M, die_of_sm=die, sched=sched),
                        iters=it)
        flops = 2.0 * M * d * V
        tok = torch.empty(M, device=dev, dtype=torch.int32)
        conf = torch.empty(M, device=dev)
        lse = torch.empty(M, device=dev)
        ms4 = timeit(lambda: hotpath.stats_merge(pm, ps, pa, S, M, M, m_host=M, token=tok, lse=lse, conf=conf))
        out[f"k3_lmhead_{name}"] = {"M": M, "d": d, "V": V, "splits": S, "tiles_per_split": tps, "ms": ms,
                                    "TFLOPs": flops / ms / 1e9, "frac_bf16_peak": flops / ms / 1e9 / tf,
                                    "schedule": "dynamic", "static_ms": ms_static,
                                    "static_TFLOPs": flops / ms_static / 1e9,
                                    "die_aware_ms": ms_die, "die_aware_TFLOPs": flops / ms_die / 1e9,
                                    "k4_merge_ms": ms4}
        del hc, W

    # K3 gather mode (gather4 A operand straight from H; K2 and Hc disappear)
    for name, L, d, V, layout in (("llada", 32768, 4096, 126464, "suffix"), ("llada_scattered", 32768, 4096, 126464,
                                                                             "scattered")):
        M = L // 2
        H = torch.randn(L, d, generator=g, device=dev).to(torch.bfloat16)
        W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
        idx = (torch.arange(L - M, L, device=dev) if layout == "suffix" else
               torch.randperm(L, generator=g, device=dev)[:M].sort().values).to(torch.int32)
        S, tps = hotpath.lmhead_plan(M, V, d)
        pm = torch.empty(S, M, device=dev)
        ps = torch.empty(S, M, device=dev)
        pa = torch.empty(S, M, device=dev, dtype=torch.int32)
        die, sched = None, torch.zeros(4, dtype=torch.int32, device=dev)  # dynamic schedule (product default)
        ms = timeit(lambda: hotpath.lmhead_stats_gather(H, idx, W, S, pm, ps, pa, M, m_host=M, die_of_sm=die,
                                                        sched=sched), iters=5)
        hc = torch.empty(M, d, device=dev, dtype=torch.bfloat16)
        ms_sep = timeit(lambda: (hotpath.gather_rows(H, idx, hc, m_host=M),
                                 hotpath.lmhead_stats(hc, W, S, pm, ps, pa, m_host=M, die_of_sm=die, sched=sched)),
                        iters=5)
        ms_runs = timeit(lambda: (hotpath.gather_rows_scattered(H, idx, hc, M, m_host=M),
                                  hotpath.lmhead_stats_runs(H, idx, hc, W, S, pm, ps, pa, M, m_host=M, die_of_sm=die,
                                                            sched=sched)), iters=5)
        flops = 2.0 * M * d * V
        out[f"k3_gather_{name}"] = {"M": M, "d": d, "V": V, "splits": S, "ms": ms, "TFLOPs": flops / ms / 1e9,
                                    "frac_bf16_peak": flops / ms / 1e9 / tf, "k2_plus_k3_ms": ms_sep,
                                    "runs_k2_plus_k3_ms": ms_runs,
                                    "schedule": "dynamic (all)", "hc_bytes_saved": M * d * 2}
        del H, W, hc

    # whole step: eager launches vs one captured CUDA graph (launch-bound at small sizes)
    from paper_2601_06562_b200 import MaskOnlyHead

    for name, L, d, V in (("tiny", 2048, 256, 8192), ("llada", 32768, 4096, 126464)):
        H = torch.randn(L, d, generator=g, device=dev).to(torch.bfloat16)
        W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
        x0 = torch.randint(0, V - 1, (L,), generator=g, device=dev, dtype=torch.int32)
        x0[L // 2:] = V - 1
        head = MaskOnlyHead(W, seq_len=L, mask_id=V - 1)
        x = x0.clone()
        eager_ms = timeit(lambda: (x.copy_(x0), head.step(x, H, 64)), iters=20)
        xg = x0.clone()
        graph = head.capture(xg, H, 64)
        graph_ms = timeit(lambda: (xg.copy_(x0), graph.replay()), iters=20)
        out[f"step_{name}"] = {"L": L, "d": d, "V": V, "eager_ms": eager_ms, "graph_ms": graph_ms}
        if name == "llada":  # semi-autoregressive block decoding: one 32-position block of the masked half
            lo = L // 2
            xw = x0.clone()
            wg = head.capture(xw, H, 4, window=(lo, lo + 32))
            win_eager = timeit(lambda: (x.copy_(x0), head.step(x, H, 4, window=(lo, lo + 32))), iters=50)
            win_graph = timeit(lambda: (xw.copy_(x0), wg.replay()), iters=50)
            out["step_llada_block32"] = {"L": L, "window": 32, "eager_ms": win_eager, "graph_ms": win_graph,
                                         "note": "step(window=(L/2, L/2+32)): K3 over <= 32 masked rows "
                                                 "streams the whole 1.04 GB LM head"}
        del H, W

    # K5 ---------------------------------------------------------------------
    for M, k in ((16384, 256), (65536, 683), (524288, 8192)):
        conf = torch.rand(M, generator=g, device=dev)
        pos = torch.arange(M, device=dev, dtype=torch.int32)
        tok = torch.zeros(M, device=dev, dtype=torch.int32)
        x = torch.zeros(M, device=dev, dtype=torch.int32)
        sc = torch.empty(hotpath.remask_scratch_bytes(), dtype=torch.uint8, device=dev)
        ms = timeit(lambda: hotpath.remask_commit(conf, pos, tok, k, x, sc, M, m_host=M))
        out[f"k5_remask_M{M}_k{k}"] = {"ms": ms}

    # K6 ---------------------------------------------------------------------
    for name, rows, f in (("llada_chunk", 32768, 12288), ("dream_chunk", 32768, 18944)):
        gate = torch.randn(rows, f, generator=g, device=dev).to(torch.bfloat16)
        up = torch.randn(rows, f, generator=g, device=dev).to(torch.bfloat16)
        ms = timeit(lambda: hotpath.swiglu_(gate, up))
        byts = 3 * 2 * rows * f
        out[f"k6_swiglu_{name}"] = {"ms": ms, "GBps": byts / ms / 1e6, "frac_hbm": byts / ms / 1e6 / hbm}
        del gate, up
    print(json.dumps(out, indent=1))
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
