"""One LLaDA-shape K3 launch in gather mode (for ncu)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_06562_b200 import hotpath, _native
_native.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
L, d, V = 32768, 4096, 126464
M = L // 2
H = torch.randn(L, d, generator=g, device=dev).to(torch.bfloat16)
W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
idx = torch.arange(L - M, L, device=dev, dtype=torch.int32)
S, _ = hotpath.lmhead_plan(M, V, d)
pm = torch.empty(S, M, device=dev); ps = torch.empty(S, M, device=dev)
pa = torch.empty(S, M, device=dev, dtype=torch.int32)
for _ in range(2):
    hotpath.lmhead_stats_gather(H, idx, W, S, pm, ps, pa, M, m_host=M)
torch.cuda.synchronize()
print("ok")
