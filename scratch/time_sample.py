"""K3 sampling variant vs argmax variant at the LLaDA head (M 16384), steady loop."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_06562_b200 import hotpath, _native
_native.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
M, d, V = 16384, 4096, 126464
hc = torch.randn(M, d, generator=g, device=dev).to(torch.bfloat16)
W = (torch.randn(V, d, generator=g, device=dev) * 0.02 * float(os.environ.get("WSCALE", "1"))).to(torch.bfloat16)
pos = torch.arange(M, dtype=torch.int32, device=dev)
S, _ = hotpath.lmhead_plan(M, V, d)
b = [torch.empty(2 * S, M, device=dev) for _ in range(4)]
pa = torch.empty(2 * S, M, device=dev, dtype=torch.int32)
die = hotpath.die_map(dev)[0]
sched = torch.zeros(4, dtype=torch.int32, device=dev)
fl = 2.0 * M * d * V
fns = {"argmax": lambda: hotpath.lmhead_stats(hc, W, S, b[0], b[1], pa, m_host=M, die_of_sm=die, sched=sched),
       "sample": lambda: hotpath.lmhead_sample(hc, W, S, pos, 1.0, 7, b[0], b[1], pa, b[2], b[3], m_host=M,
                                               die_of_sm=die, sched=sched),
       "T0.3": lambda: hotpath.lmhead_sample(hc, W, S, pos, 0.3, 7, b[0], b[1], pa, b[2], b[3], m_host=M,
                                             die_of_sm=die, sched=sched)}
for rep in range(2):
    for name, f in fns.items():
        for _ in range(10): f()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(100): f()
        e.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(e) / 100
        print(f"{name:7s} {ms:.3f} ms  {fl / ms / 1e9:.0f} TFLOP/s")
