"""Steady-state (power-capped) K3 throughput at a given shape: default vs die-aware schedule,
N back-to-back launches per config, alternating configs, CUDA events on the launch stream."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_06562_b200 import hotpath, _native
_native.load()
dev = torch.device("cuda", 0)
M, d, V = (int(a) for a in sys.argv[1:4])
n = int(sys.argv[4]) if len(sys.argv) > 4 else 200
g = torch.Generator(device=dev).manual_seed(0)
hc = torch.randn(M, d, generator=g, device=dev).to(torch.bfloat16)
W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
S, _ = hotpath.lmhead_plan(M, V, d)
pm = torch.empty(2 * S, M, device=dev); ps = torch.empty(2 * S, M, device=dev)  # room for the halves experiment
pa = torch.empty(2 * S, M, device=dev, dtype=torch.int32)
die = hotpath.die_map(dev)[0]
sched = torch.zeros(4, dtype=torch.int32, device=dev)
fl = 2.0 * M * d * V
for rep in range(2):
    for name, tab in (("default", None), ("die-aware", die)):
        for _ in range(20):
            hotpath.lmhead_stats(hc, W, S, pm, ps, pa, m_host=M, die_of_sm=tab, sched=sched)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(n):
            hotpath.lmhead_stats(hc, W, S, pm, ps, pa, m_host=M, die_of_sm=tab, sched=sched)
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / n
        print(f"M={M} d={d} V={V} {name:9s} {ms:.3f} ms  {fl / ms / 1e9:.0f} TFLOP/s")
