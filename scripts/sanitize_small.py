"""Small invocations of every kernel family for compute-sanitizer runs."""
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np, torch
import __graft_entry__ as ge
from paper_2601_06562_b200 import hotpath, MaskOnlyHead, _native
_native.load()
dev = torch.device("cuda", 0)
ge.smoke()  # K1, K2, K3 (cg2), K4, K5 at the tiny config, checked against the oracle
rng = np.random.default_rng(0)
L, d, V, mid = 3000, 256, 5000, 4999
x = rng.integers(0, V - 1, size=L).astype(np.int32); x[rng.random(L) < 0.5] = mid
H = torch.from_numpy(rng.standard_normal((L, d)).astype(np.float32)).to(dev).bfloat16()
W = torch.from_numpy((rng.standard_normal((V, d)) * 0.05).astype(np.float32)).to(dev).bfloat16()
for fg in (False, True):
    for da in (False, True):  # dynamic and dynamic die-aware unit schedules (unit ring)
        head = MaskOnlyHead(W, seq_len=L, mask_id=mid, shift=True, fused_gather=fg, die_aware=da)
        head.step(torch.from_numpy(x).to(dev), H, 50)
# runs mode with contiguous-run tiles (A boxes from H) beside scattered ones (A from the partial Hc)
xr = x.copy(); xr[500:1600] = mid
for da in (False, True):
    MaskOnlyHead(W, seq_len=L, mask_id=mid, shift=True, die_aware=da).step(torch.from_numpy(xr).to(dev), H, 50)
# windowed step and batched step (segmented K5), shift on
head = MaskOnlyHead(W, seq_len=L, mask_id=mid, shift=True)
head.step(torch.from_numpy(x).to(dev), H, 5, window=(1000, 1040))
Bx = torch.from_numpy(np.stack([x[:1000], x[1000:2000], x[2000:3000]])).to(dev)
bh = MaskOnlyHead(W, seq_len=3 * 100, mask_id=mid, shift=True)
bh.step_batch(Bx, H[:3000].reshape(3, 1000, d).contiguous(), torch.tensor([3, 0, 7], dtype=torch.int32, device=dev),
              window=(400, 500))
MaskOnlyHead(W, seq_len=3000, mask_id=mid, shift=True).step_batch(  # shift at lo = 0: rows repeat, no run tiles
    Bx, H[:3000].reshape(3, 1000, d).contiguous(), 4)
MaskOnlyHead(W, seq_len=L, mask_id=mid, temperature=0.7, seed=3).step(torch.from_numpy(x).to(dev), H, 9)
head = MaskOnlyHead(W, seq_len=L, mask_id=mid, m_cap=100)  # M <= 128 -> cta_group::1
xs = x.copy(); xs[:] = 1; xs[:90] = mid
head.step(torch.from_numpy(xs).to(dev), H, 10)
z = torch.randn(700, 64, device=dev)
n = 700 * 8
a = torch.empty(n, dtype=torch.int32, device=dev); b = torch.empty(n, dtype=torch.int32, device=dev)
w = torch.empty(n, device=dev); off = torch.empty(65, dtype=torch.int32, device=dev)
sc = torch.empty(hotpath.moe_route_scratch_bytes(700, 64), dtype=torch.uint8, device=dev)
hotpath.moe_route(z, 8, a, b, w, off, sc)
src = torch.randn(n, 256, device=dev).bfloat16(); out = torch.empty(700, 256, device=dev).bfloat16()
hotpath.moe_combine(src, b, w, 8, out)
g = torch.randn(4099 * 3, device=dev).bfloat16(); u = torch.randn(4099 * 3, device=dev).bfloat16()
hotpath.swiglu_(g, u)
# K10 dense + SwiGLU and grouped; K5 fused single-CTA path is in smoke(); the die-map probe
x = torch.randn(700, 256, device=dev).bfloat16()
wgu = (torch.randn(2 * 256, 256, device=dev) * 0.05).bfloat16()
act = torch.empty(700, 256, device=dev).bfloat16()
hotpath.ffn_gemm(x, hotpath.interleave_gate_up(wgu[:256].t().contiguous(), wgu[256:].t().contiguous()), act, 512,
                 m_host=700, swiglu=True)
wd = (torch.randn(64, 256, device=dev) * 0.05).bfloat16()
y = torch.empty(700, 64, device=dev).bfloat16()
hotpath.ffn_gemm(act, wd, y, 64, m_host=700)
offs = torch.tensor([0, 100, 100, 450, 700], dtype=torch.int32, device=dev)
wg4 = (torch.randn(4 * 512, 256, device=dev) * 0.05).bfloat16()
hotpath.ffn_gemm(x, wg4, act, 512, group_off=offs, groups=4, swiglu=True)
hotpath.die_map(dev)
torch.cuda.synchronize()
print("sanitize run ok")
