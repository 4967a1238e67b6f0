"""K10 vs cuBLAS on the FFN chunk shapes (LLaDA dense chunk, LLaDA-MoE experts)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch, torch.nn.functional as F
from paper_2601_06562_b200 import hotpath, _native
_native.load()
dev = torch.device("cuda", 0)
def t(fn, n=5):
    for _ in range(2): fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / n
M, K, Fd = 32768, 4096, 12288
x = torch.randn(M, K, device=dev).bfloat16(); wg = (torch.randn(K, Fd, device=dev) * .02).bfloat16(); wu = (torch.randn(K, Fd, device=dev) * .02).bfloat16()
wgu = hotpath.interleave_gate_up(wg, wu); act = torch.empty(M, Fd, device=dev).bfloat16()
up = torch.empty(M, Fd, device=dev).bfloat16(); gate = torch.empty(M, Fd, device=dev).bfloat16()
fl = 2 * 2 * M * K * Fd
ms_k10 = t(lambda: hotpath.ffn_gemm(x, wgu, act, 2 * Fd, m_host=M, swiglu=True))
ms_cub = t(lambda: (torch.matmul(x, wu, out=up), torch.matmul(x, wg, out=gate), hotpath.swiglu_(gate, up)))
print(f"dense gate+up+glu LLaDA chunk: K10 {ms_k10:.2f} ms ({fl/ms_k10/1e9:.0f} TF/s)  cuBLAS+K6 {ms_cub:.2f} ms ({fl/ms_cub/1e9:.0f} TF/s)")
wd = (torch.randn(Fd, K, device=dev) * .02).bfloat16(); wdt = wd.t().contiguous(); y = torch.empty(M, K, device=dev).bfloat16()
fl = 2 * M * K * Fd
ms_k10 = t(lambda: hotpath.ffn_gemm(act, wdt, y, K, m_host=M))
ms_cub = t(lambda: torch.matmul(act, wd, out=y))
print(f"dense down LLaDA chunk: K10 {ms_k10:.2f} ms ({fl/ms_k10/1e9:.0f} TF/s)  cuBLAS {ms_cub:.2f} ms ({fl/ms_cub/1e9:.0f} TF/s)")
del x, wg, wu, wgu, act, up, gate, wd, wdt, y
E, k, rows, d, Fe = 64, 8, 65536, 2048, 1408
P = rows * k
logits = torch.randn(rows, E, device=dev)
rrow = torch.empty(P, dtype=torch.int32, device=dev); rpos = torch.empty(P, dtype=torch.int32, device=dev)
rw = torch.empty(P, device=dev); off = torch.empty(E + 1, dtype=torch.int32, device=dev)
sc = torch.empty(hotpath.moe_route_scratch_bytes(rows, E), dtype=torch.uint8, device=dev)
hotpath.moe_route(logits, k, rrow, rpos, rw, off, sc)
xin = torch.randn(P, d, device=dev).bfloat16()
wg = (torch.randn(E, d, Fe, device=dev) * .02).bfloat16(); wu = (torch.randn(E, d, Fe, device=dev) * .02).bfloat16()
wgu = hotpath.interleave_gate_up(wg, wu).view(E * 2 * Fe, d); act = torch.empty(P, Fe, device=dev).bfloat16()
up = torch.empty(P, Fe, device=dev).bfloat16(); gate = torch.empty(P, Fe, device=dev).bfloat16()
o = off.cpu().tolist()
def cub():
    for e in range(E):
        if o[e + 1] > o[e]:
            torch.matmul(xin[o[e]:o[e+1]], wu[e], out=up[o[e]:o[e+1]]); torch.matmul(xin[o[e]:o[e+1]], wg[e], out=gate[o[e]:o[e+1]])
    hotpath.swiglu_(gate, up)
fl = 2 * 2 * P * d * Fe
ms_k10 = t(lambda: hotpath.ffn_gemm(xin, wgu, act, 2 * Fe, group_off=off, groups=E, swiglu=True))
ms_cub = t(cub)
print(f"MoE gate+up+glu 64x top8 64k tokens: K10 {ms_k10:.2f} ms ({fl/ms_k10/1e9:.0f} TF/s)  cuBLAS loop+K6 {ms_cub:.2f} ms ({fl/ms_cub/1e9:.0f} TF/s)")
wd = (torch.randn(E, Fe, d, device=dev) * .02).bfloat16(); wdt = wd.transpose(1, 2).contiguous().view(E * d, Fe)
y = torch.empty(P, d, device=dev).bfloat16()
def cubd():
    for e in range(E):
        if o[e + 1] > o[e]:
            torch.matmul(act[o[e]:o[e+1]], wd[e], out=y[o[e]:o[e+1]])
fl = 2 * P * d * Fe
ms_k10 = t(lambda: hotpath.ffn_gemm(act, wdt, y, d, group_off=off, groups=E))
ms_cub = t(cubd)
print(f"MoE down: K10 {ms_k10:.2f} ms ({fl/ms_k10/1e9:.0f} TF/s)  cuBLAS loop {ms_cub:.2f} ms ({fl/ms_cub/1e9:.0f} TF/s)")
