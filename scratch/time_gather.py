"""Times K3 gather mode vs K2+K3 at LLaDA shape (env selects cta_group / gather path)."""
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
hc = torch.empty(M, d, device=dev, dtype=torch.bfloat16)
def t(fn, n=5):
    for _ in range(2): fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / n
die = hotpath.die_map(dev)[0]
sched = torch.zeros(4, dtype=torch.int32, device=dev)
print("die-aware: gather %.2f ms" % t(lambda: hotpath.lmhead_stats_gather(H, idx, W, S, pm, ps, pa, M, m_host=M, die_of_sm=die, sched=sched)),
      "k2+k3 %.2f ms" % t(lambda: (hotpath.gather_rows(H, idx, hc, m_host=M), hotpath.lmhead_stats(hc, W, S, pm, ps, pa, m_host=M, die_of_sm=die, sched=sched))))
print(os.environ.get("MOSAIC_CTA_GROUP"), os.environ.get("MOSAIC_K3_GATHER"),
      "gather %.2f ms" % t(lambda: hotpath.lmhead_stats_gather(H, idx, W, S, pm, ps, pa, M, m_host=M)),
      "k2+k3 %.2f ms" % t(lambda: (hotpath.gather_rows(H, idx, hc, m_host=M), hotpath.lmhead_stats(hc, W, S, pm, ps, pa, m_host=M))))
