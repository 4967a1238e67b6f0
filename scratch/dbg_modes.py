import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
from dataclasses import replace
import numpy as np, torch
from paper_2601_06562_b200 import vmm, workload
from paper_2601_06562_b200.executor import RandomDLLM, StepExecutor
cfg = workload.toy_configs()["tiny_llada"]
dev = torch.device("cuda", 0)
model = RandomDLLM(cfg, dev, seed=3)
ws = vmm.reserve(8 << 30, backend="cuda")
ex = StepExecutor(model, ws, 8191)
L, M, k = 2048, 1024, 32
rng = np.random.default_rng(2)
x0 = rng.integers(0, 8191, size=L).astype(np.int32); x0[L-M:] = 8191
for mode in ("fused", "mask_only", "eager"):
    x = torch.from_numpy(x0).to(dev)
    t = workload.build_layer_template(replace(cfg, logits_mode=mode))
    g = t.instantiate({"L": L, "M": M, "K_logits": 1, "K_FFN": 1})
    r = ex.run(g, x, k, keep=("token_out", "l1.h_out"))
    tok = r["kept"]["token_out"]; conf = r["kept"]["confidence"]
    print(mode, tok.shape, tok[:8].tolist(), tok.min().item(), tok.max().item(), conf[:4].tolist())
    h = r["kept"]["l1.h_out"]
    z = (h[L-M:].float() @ model.w_vocab.float().t())
    print("  ref argmax", z.argmax(1)[:8].tolist())
    xo = x.cpu().numpy(); ch = np.flatnonzero(xo != x0); print("  changed", ch[:5], xo[ch[:5]])
