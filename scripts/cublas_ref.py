"""cuBLAS reference on the K3 shape (M=16384, N=126464, K=4096, bf16 out) run
back to back for ~4 s on the same box: TFLOP/s and SM clock, to separate the
box's power behaviour from the kernel's."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from bench import ClockSampler  # noqa: E402

M, N, K = 16384, 126464, 4096
a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
b = (torch.randn(N, K, device="cuda", dtype=torch.float32) * 0.02).to(torch.bfloat16)
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    torch.matmul(a, b.t(), out=out)
torch.cuda.synchronize()
n = 300
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with ClockSampler(0) as c:
    s.record()
    for _ in range(n):
        torch.matmul(a, b.t(), out=out)
    e.record()
    torch.cuda.synchronize()
ms = s.elapsed_time(e) / n
print(f"cublas {M}x{N}x{K} bf16: {ms:.3f} ms  {2*M*N*K/ms/1e9:.0f} TF  clocks={c.summary()}")
