import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_06562_b200 import MaskOnlyHead, _native
_native.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
d, V, Ls, blk, B = 4096, 126464, 2048, 32, 64
W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
H = torch.randn(B, Ls, d, generator=g, device=dev).to(torch.bfloat16)
x0 = torch.randint(0, V - 1, (B, Ls), generator=g, device=dev, dtype=torch.int32)
lo = Ls // 2
x0[:, lo:] = V - 1
head = MaskOnlyHead(W, seq_len=B * blk, mask_id=V - 1)
x = x0.clone(); xg = x0.clone()
graph = head.capture(xg, H, 4, window=(lo, lo + blk))
mode = sys.argv[1]
for _ in range(6):
    if mode == "eager":
        x.copy_(x0); head.step_batch(x, H, 4, window=(lo, lo + blk))
    else:
        xg.copy_(x0); graph.replay()
torch.cuda.synchronize()
