"""K5 remask commit: single-CTA fused path vs the multi-launch radix select, by M."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_06562_b200 import hotpath, _native
_native.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
for M in (4096, 8192, 16384, 24576, 32768, 49152, 65536):
    conf = torch.rand(M, generator=g, device=dev) * 1e-3 + 1e-4
    pos = torch.arange(M, device=dev, dtype=torch.int32) * 2
    tok = torch.randint(0, 1000, (M,), generator=g, device=dev, dtype=torch.int32)
    x = torch.zeros(2 * M, dtype=torch.int32, device=dev)
    sc = torch.empty(hotpath.remask_scratch_bytes(), dtype=torch.uint8, device=dev)
    k = max(1, M // 64)
    f = lambda: hotpath.remask_commit(conf, pos, tok, k, x, sc, M, m_host=M)
    for _ in range(5): f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(50): f()
    b.record(); torch.cuda.synchronize()
    print(f"M={M} cap={os.environ.get('MOSAIC_K5_FUSED_CAP', 'default')} {a.elapsed_time(b) / 50 * 1e3:.1f} us")
