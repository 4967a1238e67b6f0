"""Plain-PyTorch references for the step executor's numerics (test
infrastructure: no arena, no chunking, no hand-written kernels).

``reference_forward`` runs the same random-init model as
``paper_2601_06562_b200.executor.RandomDLLM`` layer by layer with torch ops and
returns the final hidden states the executor's in-arena forward must match.
"""
from __future__ import annotations

import torch
import torch.nn.functional as F

from paper_2601_06562_b200.executor import RandomDLLM
from paper_2601_06562_b200.workload import ModelConfig


def reference_forward(model: RandomDLLM, x: torch.Tensor) -> torch.Tensor:
    """Plain-PyTorch forward of the same model (no arena, no chunking): the
    final hidden states [L, d], used as the executor's numerics reference."""
    cfg = model.cfg
    L, d, H = x.numel(), cfg.d_model, cfg.n_heads
    h = model.w_embed.index_select(0, x)
    for i in range(cfg.n_layers):
        lw = model.layer(i)
        q, k, v = (h @ lw["w_qkv"][:, j * d:(j + 1) * d] for j in range(3))
        if model.inv_freq is not None:
            q, k = rope(q, H, model.inv_freq), rope(k, H, model.inv_freq)
        qh, kh, vh = (t.view(L, H, d // H).transpose(0, 1).unsqueeze(0) for t in (q, k, v))
        a = F.scaled_dot_product_attention(qh, kh, vh).squeeze(0).transpose(0, 1).reshape(L, d)
        h = h + a @ lw["w_attn_out"]
        if cfg.moe is not None:
            h = h + _moe_reference(cfg, lw, h)
            continue
        if "w_gate_up" in lw:  # fused_ffn layout -> torch layout
            wg, wu = _split_gate_up(lw["w_gate_up"], cfg.d_ff)
            lw = {**lw, "w_gate": wg, "w_up": wu, "w_down": lw["w_down"].t()}  # K-major [d, f] -> [f, d]
        up = h @ lw["w_up"]
        act = F.silu((h @ lw["w_gate"]).float()).mul(up.float()).to(torch.bfloat16) if cfg.gated_ffn else F.silu(up)
        h = h + act @ lw["w_down"]
    return h


def rope(t: torch.Tensor, n_heads: int, inv_freq: torch.Tensor) -> torch.Tensor:
    """Rotate-half rotary embedding of [L, n_heads * dh] bf16 rows in fp32 math
    (the rule K11 applies in place), rounded back to bf16."""
    L, d = t.shape
    dh = d // n_heads
    ang = torch.arange(L, device=t.device, dtype=torch.float32)[:, None] * inv_freq[None, :]  # [L, dh/2]
    c, s = torch.cos(ang)[:, None, :], torch.sin(ang)[:, None, :]
    x = t.view(L, n_heads, dh).float()
    a, b = x[..., : dh // 2], x[..., dh // 2:]
    return torch.cat([a * c - b * s, b * c + a * s], dim=-1).to(torch.bfloat16).view(L, d)


def _moe_reference(cfg: ModelConfig, lw: dict, h: torch.Tensor) -> torch.Tensor:
    """Plain-PyTorch MoE FFN with the routing rule of K8: top-k by (logit desc,
    expert asc) over fp32 router logits, softmax over the selected logits,
    per-expert SwiGLU FFN, weighted fp32 sum."""
    E, k = cfg.moe.n_experts, cfg.moe.top_k
    d, f = cfg.d_model, cfg.d_ff
    wg, wu = _split_gate_up(lw["w_gate_up"].view(E, 2 * f, d), f)              # [E, d, f] each
    wd = lw["w_down"].view(E, d, f).transpose(1, 2)                           # [E, f, d]
    logits = torch.mm(h, lw["w_router"], out_dtype=torch.float32)
    vals, idx = torch.sort(logits, dim=1, descending=True, stable=True)
    sel, wts = idx[:, :k], torch.softmax(vals[:, :k], dim=1)
    out = torch.zeros(h.shape, dtype=torch.float32, device=h.device)
    for e in range(E):
        rows, j = (sel == e).nonzero(as_tuple=True)
        if rows.numel() == 0:
            continue
        x = h.index_select(0, rows)
        up = x @ wu[e]
        act = F.silu((x @ wg[e]).float()).mul(up.float()).to(torch.bfloat16)
        out.index_add_(0, rows, wts[rows, j].unsqueeze(1) * (act @ wd[e]).float())
    return out.to(torch.bfloat16)


def _split_gate_up(w_gu: torch.Tensor, f: int) -> tuple[torch.Tensor, torch.Tensor]:
    """Inverse of hotpath.interleave_gate_up: [.., 2f, d] -> gate, up [.., d, f]."""
    *lead, _, d = w_gu.shape
    blocks = w_gu.reshape(*lead, f // 128, 2, 128, d)
    gate = blocks[..., 0, :, :].reshape(*lead, f, d).transpose(-1, -2)
    up = blocks[..., 1, :, :].reshape(*lead, f, d).transpose(-1, -2)
    return gate, up
