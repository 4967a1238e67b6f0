"""Vocab-sharded LM head across the GPUs of one box (north_star item 4).

Rank r of P holds the contiguous vocab slice [r*V//P, (r+1)*V//P) of the LM
head. After K3+K4 each rank has one (max, sum-exp, argmax) triple per masked
row for its slice (argmax already carries the global vocab id via the
shard's offset); the only exchange is an all-gather of those triples — 12
bytes per row per rank over NVLink — after which every rank merges the P
triples in rank order (K4) and runs the identical, deterministic remask
(K5). Mask compaction, gather and the rest of the step are replicated.

The reference has no distribution; rows are independent
(mosaic/kernel.py:70-84) and the triple merge is associative, which is what
makes this exact.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def vocab_shard_bounds(vocab: int, world: int, rank: int) -> tuple[int, int]:
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    return rank * vocab // world, (rank + 1) * vocab // world


def exchange_triples(local: torch.Tensor, group=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather a [3, m] fp32 triple block (max, sum, argmax bits) into
    [P, 3, m], rank-major, so that K4 can merge it with stride 3*m."""
    if local.dim() != 2 or local.shape[0] != 3 or local.dtype != torch.float32:
        raise ValueError("local triples must be fp32 [3, m]")
    world = dist.get_world_size(group)
    if out is None:
        out = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
    backend = dist.get_backend(group)
    if backend == "nccl":
        dist.all_gather_into_tensor(out.view(-1), local.contiguous().view(-1), group=group)
    else:  # gloo (CPU tests): list form
        parts = list(out.unbind(0))
        dist.all_gather(parts, local.contiguous(), group=group)
    return out


def pack_triples(mx: torch.Tensor, sm: torch.Tensor, arg: torch.Tensor) -> torch.Tensor:
    """[3, m] fp32 block with the int32 argmax stored bit-exactly in row 2."""
    out = torch.empty((3, mx.numel()), dtype=torch.float32, device=mx.device)
    out[0].copy_(mx)
    out[1].copy_(sm)
    out[2].view(torch.int32).copy_(arg.to(torch.int32))
    return out


def unpack_triples(block: torch.Tensor):
    """Inverse of :func:`pack_triples` for a [..., 3, m] block."""
    return block[..., 0, :], block[..., 1, :], block[..., 2, :].contiguous().view(torch.int32)
