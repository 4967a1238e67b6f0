"""Same-box A/B of K10's static vs dynamic tile schedule on the LLaDA 32k FFN
chunk GEMMs (gate/up + SwiGLU: 32768 x 4096 -> 2 x 12288; down + residual:
32768 x 12288 -> 4096) and the Dream 128k chunk (K = 3584 / 18944),
alternating, CUDA events.   python scripts/k10_sched_ab.py [--reps 3]"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    from paper_2601_06562_b200 import _build, hotpath

    _build.build()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    sched = torch.zeros(4, dtype=torch.int32, device=dev)
    for name, M, d, f in (("llada", 32768, 4096, 12288), ("dream", 32768, 3584, 18944)):
        x = torch.randn(M, d, generator=g, device=dev).to(torch.bfloat16)
        wgu = (torch.randn(2 * f, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
        wd = (torch.randn(d, f, generator=g, device=dev) * 0.02).to(torch.bfloat16)
        act = torch.empty(M, f, device=dev, dtype=torch.bfloat16)
        res = {}
        for op in ("gate_up", "down"):
            flops = 2.0 * M * d * (2 * f if op == "gate_up" else f)
            for mode in ("static", "dynamic"):
                res.setdefault(f"{op}_{mode}", [])
            for _ in range(a.reps):
                for mode in ("static", "dynamic"):
                    kw = dict(sched=sched) if mode == "dynamic" else {}

                    def run():
                        if op == "gate_up":
                            hotpath.ffn_gemm(x, wgu, act, 2 * f, m_host=M, swiglu=True, **kw)
                        else:
                            hotpath.ffn_gemm(act, wd, x, d, m_host=M, residual=True, **kw)

                    for _ in range(2):
                        run()
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    s.record()
                    for _ in range(10):
                        run()
                    e.record()
                    e.synchronize()
                    res[f"{op}_{mode}"].append(round(flops / (s.elapsed_time(e) / 10) / 1e9, 1))
        print(json.dumps({"shape": name, "M": M, "d": d, "d_ff": f, "tflops": res}), flush=True)
        del x, wgu, wd, act


if __name__ == "__main__":
    main()
