import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np, torch
from paper_2601_06562_b200 import MaskOnlyHead, _native
_native.load()
dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)
L, d, V, mid = 3000, 256, 5000, 4999
x = rng.integers(0, V - 1, size=L).astype(np.int32); x[rng.random(L) < 0.5] = mid
H = torch.from_numpy(rng.standard_normal((L, d)).astype(np.float32)).to(dev).bfloat16()
W = torch.from_numpy((rng.standard_normal((V, d)) * 0.05).astype(np.float32)).to(dev).bfloat16()
MaskOnlyHead(W, seq_len=L, mask_id=mid, temperature=0.7, seed=3).step(torch.from_numpy(x).to(dev), H, 9)
torch.cuda.synchronize(); print("ok")
