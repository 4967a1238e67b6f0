"""Batched block decoding: B sequences x one 32-position block, LLaDA head, one
step_batch vs B windowed steps."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_06562_b200 import MaskOnlyHead, _native
_native.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
d, V, Ls, blk = 4096, 126464, 2048, 32
W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
for B in (1, 8, 32, 64, 128):
    H = torch.randn(B, Ls, d, generator=g, device=dev).to(torch.bfloat16)
    x0 = torch.randint(0, V - 1, (B, Ls), generator=g, device=dev, dtype=torch.int32)
    x0[:, Ls // 2:] = V - 1
    lo = Ls // 2
    head = MaskOnlyHead(W, seq_len=B * blk, mask_id=V - 1)
    one = MaskOnlyHead(W, seq_len=Ls, mask_id=V - 1)
    x = x0.clone()
    def batched():
        x.copy_(x0); head.step_batch(x, H, 4, window=(lo, lo + blk))
    def looped():
        x.copy_(x0)
        for b in range(B):
            one.step(x[b], H[b], 4, window=(lo, lo + blk))
    res = []
    for f in (batched, looped):
        for _ in range(3): f()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record()
        for _ in range(10): f()
        e.record(); torch.cuda.synchronize()
        res.append(a.elapsed_time(e) / 10)
    print(f"B={B:4d} block={blk}: step_batch {res[0]:.3f} ms  ({B * blk / res[0] * 1e3 / 1e6:.2f} M masked tok/s)   "
          f"B windowed steps {res[1]:.3f} ms")
