"""Parity of the pre-tiled W experiment: one fused step, hash of the outputs (run with and without
MOSAIC_K3_WBLOCKED=1; the hashes must match)."""
import os, sys, hashlib
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_06562_b200 import MaskOnlyHead, _native
_native.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(5)
L, D, V = 8192, 4096, 126464
W = (torch.randn(V, D, generator=g, device=dev) * 0.02).to(torch.bfloat16)
H = torch.randn(L, D, generator=g, device=dev).to(torch.bfloat16)
x = torch.randint(0, V - 1, (L,), generator=g, device=dev, dtype=torch.int32)
x[L // 2:] = V - 1
if os.environ.get("MOSAIC_K3_WBLOCKED") == "1":
    n_t = -(-V // 256)
    W = W.view(n_t, 256, D // 64, 64).permute(0, 2, 1, 3).contiguous().view(n_t * 256, D)
head = MaskOnlyHead(W, seq_len=L, mask_id=V - 1)
o = head.step(x, H, 100)
torch.cuda.synchronize()
M = int(o.m_dev.item())
h = hashlib.sha1()
for t in (o.token[:M], o.conf[:M], o.lse[:M], x):
    h.update(t.cpu().numpy().tobytes())
print("hash", os.environ.get("MOSAIC_K3_WBLOCKED", "0"), h.hexdigest())
