"""One launch each of the HBM-bound kernels (K2 gather, K6 SwiGLU, K9 combine,
K11 RoPE) and of K10 (FFN GEMM: gate/up + SwiGLU, down + residual) at the
BASELINE shapes, for an ncu --set full capture:
    ncu --set full -k regex:'k2_|k6_|k9_|k10_|k11_' -o prof python scripts/ncu_targets.py
K2 runs on a scattered layout (every tile gathered: runs mode compacts all rows,
the same launch the buffered path makes)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

from paper_2601_06562_b200 import _native, hotpath

_native.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
# K2: LLaDA 32k, 16384 masked rows of d 4096
L, d = 32768, 4096
H = torch.randn(L, d, generator=g, device=dev).to(torch.bfloat16)
idx = torch.randperm(L, generator=g, device=dev)[: L // 2].sort().values.to(torch.int32)
hc = torch.empty(L // 2, d, device=dev, dtype=torch.bfloat16)
hotpath.gather_rows_scattered(H, idx, hc, L // 2, m_host=L // 2)
# K11: rotary positions on q and k of one LLaDA layer at 32k (32 heads of 128)
q = torch.randn(L, d, generator=g, device=dev).to(torch.bfloat16)
inv = hotpath.rope_inv_freq(128, 10000.0, dev)
hotpath.rope_qk_(q, H, 32, inv)
del H, hc, q
# K6: LLaDA FFN chunk 32768 x 12288
gate = torch.randn(32768, 12288, generator=g, device=dev).to(torch.bfloat16)
up = torch.randn(32768, 12288, generator=g, device=dev).to(torch.bfloat16)
hotpath.swiglu_(gate, up)
del gate, up
# K9: MoE combine, 65536 tokens x top-8, d 2048
rows, k, dm = 65536, 8, 2048
src = torch.randn(rows * k, dm, generator=g, device=dev).to(torch.bfloat16)
pos = torch.randperm(rows * k, generator=g, device=dev).to(torch.int32)
w = torch.rand(rows * k, generator=g, device=dev)
out = torch.empty(rows, dm, device=dev, dtype=torch.bfloat16)
hotpath.moe_combine(src, pos, w, k, out)
del src, out
# K10: dense gate/up + SwiGLU on the LLaDA chunk
x = torch.randn(32768, 4096, generator=g, device=dev).to(torch.bfloat16)
wgu = (torch.randn(2 * 12288, 4096, generator=g, device=dev) * 0.02).to(torch.bfloat16)
act = torch.empty(32768, 12288, device=dev, dtype=torch.bfloat16)
sched = torch.zeros(4, dtype=torch.int32, device=dev)  # the dynamic tile schedule the executor uses
hotpath.ffn_gemm(x, wgu, act, 2 * 12288, m_host=32768, swiglu=True, sched=sched)
# K10: dense down projection with the residual epilogue (h[rows] += act @ W_down)
wd = (torch.randn(4096, 12288, generator=g, device=dev) * 0.02).to(torch.bfloat16)
hotpath.ffn_gemm(act, wd, x, 4096, m_host=32768, residual=True, sched=sched)
torch.cuda.synchronize()
print("ok")
