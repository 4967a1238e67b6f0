"""K6 bandwidth and Dream-shape K3 schedule knobs (env) on one B200."""
import sys, os, json
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_06562_b200 import hotpath, _native
_native.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
def t(fn, n=10):
    for _ in range(3): fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / n
if os.environ.get("WHAT", "k6") == "k6":
    for rows, f in ((32768, 12288), (32768, 18944), (1000, 1001)):
        gate = torch.randn(rows, f, generator=g, device=dev).to(torch.bfloat16)
        up = torch.randn(rows, f, generator=g, device=dev).to(torch.bfloat16)
        ms = t(lambda: hotpath.swiglu_(gate, up))
        print(f"k6 {rows}x{f}: {ms:.3f} ms {6 * rows * f / ms / 1e6:.0f} GB/s")
        del gate, up
else:
    M, d, V = 65536, 3584, 152064
    hc = torch.randn(M, d, generator=g, device=dev).to(torch.bfloat16)
    W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
    S, tps = hotpath.lmhead_plan(M, V, d)
    pm = torch.empty(S, M, device=dev); ps = torch.empty(S, M, device=dev)
    pa = torch.empty(S, M, device=dev, dtype=torch.int32)
    ms = t(lambda: hotpath.lmhead_stats(hc, W, S, pm, ps, pa, m_host=M), n=5)
    print(f"dream K3 gm={os.environ.get('MOSAIC_GROUP_M')} tps={tps} S={S}: {ms:.2f} ms {2*M*d*V/ms/1e9:.0f} TF/s")
