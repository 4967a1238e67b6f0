"""One small K3 launch per A path under compute-sanitizer racecheck (full hazard
detail): python scripts/racecheck_k3.py [buffered|runs|k10]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_06562_b200 import _native, hotpath  # noqa: E402

_native.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
mode = sys.argv[1] if len(sys.argv) > 1 else "runs"
M, d, V = 1024, 256, 4096
H = torch.randn(4096, d, generator=g, device=dev).to(torch.bfloat16)
W = (torch.randn(V, d, generator=g, device=dev) * 0.05).to(torch.bfloat16)
idx = torch.arange(1000, 1000 + M, device=dev, dtype=torch.int32)
S, _ = hotpath.lmhead_plan(M, V, d)
pm, ps = torch.empty(S, M, device=dev), torch.empty(S, M, device=dev)
pa = torch.empty(S, M, dtype=torch.int32, device=dev)
hc = torch.empty(M, d, dtype=torch.bfloat16, device=dev)
if mode == "buffered":
    hotpath.gather_rows(H, idx, hc, m_host=M)
    hotpath.lmhead_stats(hc, W, S, pm, ps, pa, m_host=M)
elif mode == "runs":
    hotpath.gather_rows_scattered(H, idx, hc, M, m_host=M)
    hotpath.lmhead_stats_runs(H, idx, hc, W, S, pm, ps, pa, M, m_host=M)
else:
    out = torch.empty(M, 512, dtype=torch.bfloat16, device=dev)
    hotpath.ffn_gemm(hc, (torch.randn(512, d, generator=g, device=dev) * 0.05).to(torch.bfloat16), out, 512, m_host=M)
torch.cuda.synchronize()
print("ok", mode)
