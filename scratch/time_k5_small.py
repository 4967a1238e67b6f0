"""K5 at small row counts (rank-count vs radix threshold)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_06562_b200 import hotpath, _native
_native.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
for M in (32, 128, 256, 257, 512, 1024):
    conf = torch.rand(M, generator=g, device=dev) * 1e-3 + 1e-4
    pos = torch.arange(M, device=dev, dtype=torch.int32) * 2
    tok = torch.randint(0, 1000, (M,), generator=g, device=dev, dtype=torch.int32)
    x = torch.zeros(2 * M, dtype=torch.int32, device=dev)
    sc = torch.empty(hotpath.remask_scratch_bytes(), dtype=torch.uint8, device=dev)
    f = lambda: hotpath.remask_commit(conf, pos, tok, max(1, M // 8), x, sc, M, m_host=M)
    for _ in range(5): f()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(20): f()
    gr.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); gr.replay(); b.record(); torch.cuda.synchronize()
    print(f"M={M} K5 {a.elapsed_time(b) / 20 * 1e3:.1f} us")
