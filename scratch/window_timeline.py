import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_06562_b200 import MaskOnlyHead, _native
_native.load()
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
d, V, L = 4096, 126464, 32768
W = (torch.randn(V, d, generator=g, device=dev) * 0.02).to(torch.bfloat16)
H = torch.randn(L, d, generator=g, device=dev).to(torch.bfloat16)
x0 = torch.randint(0, V - 1, (L,), generator=g, device=dev, dtype=torch.int32)
x0[L // 2:] = V - 1
head = MaskOnlyHead(W, seq_len=L, mask_id=V - 1)
x = x0.clone()
graph = head.capture(x, H, 4, window=(L // 2, L // 2 + 32))
for _ in range(5):
    x.copy_(x0); graph.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    graph.replay()
b.record(); torch.cuda.synchronize()
print("graph replay ms", a.elapsed_time(b) / 50)
