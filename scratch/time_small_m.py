"""K3 (+K4) time at small masked counts (semi-autoregressive block decoding),
LLaDA head (d 4096, V 126464): latency- and W-bandwidth-bound regime."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_06562_b200 import hotpath, _native
_native.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
d, V = 4096, 126464
W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
if os.environ.get("MOSAIC_K3_WBLOCKED") == "1":  # pre-tiled W experiment (V is a multiple of 256 here)
    W = W.view(V // 256, 256, d // 64, 64).permute(0, 2, 1, 3).contiguous().view(V, d)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
for M in (1, 8, 32, 64, 128, 256, 512, 1024):
    hc = torch.randn(M, d, generator=g, device=dev).to(torch.bfloat16)
    S, tps = hotpath.lmhead_plan(M, V, d)
    pm = torch.empty(S, M, device=dev); ps = torch.empty(S, M, device=dev)
    pa = torch.empty(S, M, device=dev, dtype=torch.int32)
    tok = torch.empty(M, device=dev, dtype=torch.int32); lse = torch.empty(M, device=dev); conf = torch.empty(M, device=dev)
    def step():
        hotpath.lmhead_stats(hc, W, S, pm, ps, pa, m_host=M)
        hotpath.stats_merge(pm, ps, pa, S, M, M, m_host=M, token=tok, lse=lse, conf=conf)
    for _ in range(3): step()
    ts = []
    for _ in range(20):
        flush.zero_()  # W out of L2: the cold-W case of a real step
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); step(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    ms = ts[len(ts) // 2]
    print(f"M={M:5d} S={S:3d} tps={tps:3d}  K3+K4 {ms*1e3:7.1f} us  W stream {2*V*d/ms/1e6:6.0f} GB/s  {2*M*d*V/ms/1e9:7.1f} TFLOP/s")
