"""One gather-mode K3 step (cp.async A path, pair tiles) and one buffered step,
small, for a full-detail compute-sanitizer racecheck report."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from paper_2601_06562_b200 import MaskOnlyHead, _native

_native.load()
dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)
L, d, V, mid = 3000, 256, 5000, 4999
x = rng.integers(0, V - 1, size=L).astype(np.int32)
x[rng.random(L) < 0.5] = mid
H = torch.from_numpy(rng.standard_normal((L, d)).astype(np.float32)).to(dev).bfloat16()
W = torch.from_numpy((rng.standard_normal((V, d)) * 0.05).astype(np.float32)).to(dev).bfloat16()
mode = sys.argv[1] if len(sys.argv) > 1 else "gather"
head = MaskOnlyHead(W, seq_len=L, mask_id=mid, fused_gather=(mode == "gather"), die_aware=False)
head.step(torch.from_numpy(x).to(dev), H, 50)
torch.cuda.synchronize()
print("sanitize run ok", mode)
