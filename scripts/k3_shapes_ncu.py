"""One K3 launch at the LLaDA (configs[1]) and Dream (configs[2]) head shapes
for an ncu comparison; MOSAIC_K3_MODE = static | dynamic | die (default die):
    ncu --set full -k regex:k3_lmhead -c 2 -o prof python scripts/k3_shapes_ncu.py"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_2601_06562_b200 import _native, hotpath

_native.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
table, _ = hotpath.die_map(dev)
sched = torch.zeros(4, dtype=torch.int32, device=dev)
for M, d, V in ((16384, 4096, 126464), (65536, 3584, 152064)):
    hc = torch.randn(M, d, generator=g, device=dev).to(torch.bfloat16)
    W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
    S, _ = hotpath.lmhead_plan(M, V, d)
    pm, ps = torch.empty(S, M, device=dev), torch.empty(S, M, device=dev)
    pa = torch.empty(S, M, device=dev, dtype=torch.int32)
    mode = os.environ.get("MOSAIC_K3_MODE", "die")
    kw = {} if mode == "static" else dict(sched=sched) if mode == "dynamic" else dict(die_of_sm=table, sched=sched)
    hotpath.lmhead_stats(hc, W, S, pm, ps, pa, m_host=M, **kw)
    torch.cuda.synchronize()
    del hc, W
print("ok")
