"""Per-box A/B of K3's default vs die-aware schedule: short bursts (autotune candidate) vs steady loops."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_06562_b200 import hotpath, _native
_native.load()
dev = torch.device("cuda", 0)
M, d, V = (int(a) for a in sys.argv[1:4])
g = torch.Generator(device=dev).manual_seed(0)
hc = torch.randn(M, d, generator=g, device=dev).to(torch.bfloat16)
W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
S, _ = hotpath.lmhead_plan(M, V, d)
pm = torch.empty(S, M, device=dev); ps = torch.empty(S, M, device=dev)
pa = torch.empty(S, M, device=dev, dtype=torch.int32)
die = hotpath.die_map(dev)[0]
sched = torch.zeros(4, dtype=torch.int32, device=dev)
def run(tab, n):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(n):
        hotpath.lmhead_stats(hc, W, S, pm, ps, pa, m_host=M, die_of_sm=tab, sched=sched)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
for label, n, reps in (("burst", 20, 3), ("steady", 300, 2)):
    res = {"default": [], "die": []}
    for _ in range(reps):
        for name, tab in (("default", None), ("die", die)):
            res[name].append(run(tab, n))
    print(label, {k: [round(x, 3) for x in v] for k, v in res.items()},
          "die-aware gain %.1f%%" % (100 * (sum(res["default"]) / sum(res["die"]) - 1)))
