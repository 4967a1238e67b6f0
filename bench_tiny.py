"""BASELINE.json configs[0]: the tiny LLaDA-style dLLM (2 layers, d 256, d_ff
768, V 8192, random-init) at seq 2048 with 50% masked -- the one config the
reference's CPU path can run in full. One denoising step on the B200 (forward
in the cuMem arena + the fused K1-K5 hot path, and the hot path alone as a
captured CUDA graph) beside the reference algorithm on the host: the oracle
restatement of gather_gemm (mosaic/kernel.py:62-86, tiles 128, fp64) over all
1024 masked rows of the same final hidden states, then the softmax statistics
and the remask -- with the two results compared.

    python bench_tiny.py [--out FILE]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MASK_ID = 8191


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    from paper_2601_06562_b200 import MaskOnlyHead, _build, vmm, workload
    from paper_2601_06562_b200.executor import RandomDLLM, StepExecutor

    _build.build()
    dev = torch.device("cuda", 0)
    cfg = workload.toy_configs()["tiny_llada"]
    L, M, k = 2048, 1024, 64
    model = RandomDLLM(cfg, dev, seed=3)
    ws = vmm.reserve(1 << 30, backend="cuda")
    ex = StepExecutor(model, ws, MASK_ID)
    rng = np.random.default_rng(0)
    x0 = rng.integers(0, MASK_ID, size=L).astype(np.int32)
    x0[L - M:] = MASK_ID
    g = workload.build_layer_template(cfg).instantiate({"L": L, "M": M, "K_logits": 1, "K_FFN": 1})
    for _ in range(3):
        ex.run(g, torch.from_numpy(x0).to(dev), k)
    times = []
    for _ in range(20):
        xd = torch.from_numpy(x0).to(dev)
        r = ex.run(g, xd, k, keep=("l1.h_out",))
        times.append(r["ms"])
    step_ms = float(np.median(times))
    h = r["kept"]["l1.h_out"]
    x_gpu = xd.cpu().numpy()

    # hot path alone as one CUDA graph over the same final hidden states
    head = MaskOnlyHead(model.w_vocab, seq_len=L, mask_id=MASK_ID)
    xg = torch.from_numpy(x0).to(dev)
    graph = head.capture(xg, h, k)
    graph.replay()
    torch.cuda.synchronize()
    x_head = xg.cpu().numpy()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(100):
        xg.copy_(torch.from_numpy(x0).to(dev, non_blocking=True))
        graph.replay()
    ev1.record()
    torch.cuda.synchronize()
    hot_graph_ms = ev0.elapsed_time(ev1) / 100

    # the reference algorithm on the host, same final hidden states
    sys.path.insert(0, str(ROOT / "oracle"))
    import mosaic_oracle as orc

    H = h.float().cpu().numpy().astype(np.float64)
    W_dv = model.w_vocab.float().cpu().numpy().astype(np.float64).T
    idx = orc.mask_compact(x0, MASK_ID)
    t0 = time.perf_counter()
    logits = orc.gather_gemm(H, W_dv, tuple(int(i) for i in idx), 128, 128, 128)
    st = orc.softmax_stats(logits)
    sel = orc.remask_select(st["conf"], idx, k)
    cpu_s = time.perf_counter() - t0
    t_ref_gemm = time.perf_counter()
    orc.gather_gemm(H, W_dv, tuple(int(i) for i in idx), 128, 128, 128)
    cpu_gemm_s = time.perf_counter() - t_ref_gemm
    x_cpu = orc.commit(x0, idx, st["arg"], sel)

    # the reference operator itself through the drop-in API: numpy in, numpy
    # [M, V] logits out (host copies included), as mosaic.kernel.gather_gemm
    from paper_2601_06562_b200 import GatherGemmProblem, gather_gemm
    prob = GatherGemmProblem(H.astype(np.float32), W_dv.astype(np.float32), tuple(int(i) for i in idx))
    gather_gemm(prob)
    torch.cuda.synchronize()
    t_api = time.perf_counter()
    n_api = 20
    for _ in range(n_api):
        out_api, _ = gather_gemm(prob)
    api_s = (time.perf_counter() - t_api) / n_api
    api_err = float(np.max(np.abs(out_api.astype(np.float64) - logits)) / np.max(np.abs(logits)))
    tok_gpu = head.buf["token"][:M].cpu().numpy()
    conf_gpu = head.buf["conf"][:M].cpu().numpy()
    lse_gpu = head.buf["lse"][:M].cpu().numpy()
    ok = st["margin"] > 1e-3
    sel_gpu = (x_head != MASK_ID)[idx]
    line = {
        "workload": "tiny_llada_2k_mask50",
        "config": {"n_layers": 2, "d_model": 256, "d_ff": 768, "vocab": 8192, "seq_len": L, "masked": M,
                   "unmask_k": k},
        "gpu_step_ms": step_ms, "gpu_hot_path_graph_ms": hot_graph_ms,
        "gpu_masked_tokens_per_s_hot_path": M / (hot_graph_ms / 1e3),
        "cpu_reference_hot_path_s": cpu_s, "cpu_masked_tokens_per_s": M / cpu_s,
        "cpu_cores": len(os.sched_getaffinity(0)), "cpu_kind": "port (oracle restatement of gather_gemm, tiles 128, fp64)",
        "drop_in_gather_gemm": {"gpu_api_s": api_s, "cpu_reference_algorithm_s": cpu_gemm_s,
                                "speedup": cpu_gemm_s / api_s, "max_abs_err_rel_to_max_logit": api_err,
                                "note": "GatherGemmProblem(fp32 numpy H [2048,256], W [256,8192], 1024 idx) -> "
                                        "numpy [1024, 8192] logits, host<->device copies inside; CPU = the "
                                        "reference's tile loop (oracle restatement, tiles 128, fp64)"},
        "head_graph_equals_executor": bool(np.array_equal(x_head, x_gpu)),
        "tokens_equal_where_margin_gt_1e-3": bool(np.array_equal(tok_gpu[ok], st["arg"][ok])),
        "rows_with_margin_gt_1e-3": int(ok.sum()),
        "lse_max_rel_err": float(np.max(np.abs(lse_gpu - st["lse"]) / np.abs(st["lse"]))),
        "conf_max_rel_err": float(np.max(np.abs(conf_gpu - st["conf"]) / st["conf"])),
        "selection_equals_rule_on_device_conf": bool(np.array_equal(sel_gpu, orc.remask_select(conf_gpu, idx, k))),
        "selection_vs_fp64": orc.selection_parity(sel_gpu, conf_gpu, st["conf"], idx, k, 1e-6),
    }
    print(json.dumps(line), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(line, indent=1))
    ws.close()


if __name__ == "__main__":
    main()
