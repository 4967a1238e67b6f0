"""Control for compute-sanitizer racecheck: one cuBLAS bf16 GEMM (tcgen05 /
TMA kernels on B200, not this library's). If racecheck reports hazards at an
unattributed PC there too, the same reports in K3 / K10 are the tool's view of
the hardware's asynchronous shared-memory writes, not a race in our code.

    compute-sanitizer --tool racecheck python scripts/racecheck_cublas.py
"""
import torch

a = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
b = torch.randn(4096, 4096, device="cuda", dtype=torch.bfloat16)
c = a @ b
torch.cuda.synchronize()
print("cublas gemm ok", float(c.float().abs().mean()))
