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


class P2PExchange:
    """The exchange fused into the split merge over NVLink peer memory (K4x,
    csrc/exchange.cu): symmetric ``gathered`` [2, P, 3, m] fp32 (double-buffered
    by epoch parity) and ``signal`` [P] uint32 buffers (torch symmetric memory),
    their peers' device pointers, and a per-step epoch. ``push`` merges this
    rank's S split triples per row and stores them into every rank's gathered
    slot [epoch & 1, rank], then signals; ``wait`` blocks the stream until every
    rank has signalled this epoch; :attr:`current` is the half to merge. No
    NCCL call on the step path."""

    def __init__(self, m_cap: int, group, device):
        import torch.distributed._symmetric_memory as symm_mem

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        gathered = symm_mem.empty((2, world, 3, int(m_cap)), dtype=torch.float32, device=device)
        signal = symm_mem.empty((world,), dtype=torch.int32, device=device)
        signal.zero_()
        torch.cuda.synchronize(device)
        hg = symm_mem.rendezvous(gathered, group)
        hs = symm_mem.rendezvous(signal, group)
        self._init(gathered, signal, list(hg.buffer_ptrs), list(hs.buffer_ptrs), rank, world)
        dist.barrier(group)  # every rank's pads are zero before anyone signals

    @classmethod
    def ipc(cls, m_cap: int, group, device) -> "P2PExchange":
        """The same exchange with the peer buffers mapped through CUDA IPC
        handles traded over the process group (torch.multiprocessing's tensor
        reductions) instead of symmetric memory -- for ranks that share one GPU
        (symmetric memory refuses overlapping devices), e.g. the multi-rank
        bench test on a one-GPU box. The data path (csrc/exchange.cu) is the
        same peer-pointer stores and signal pads."""
        from torch.multiprocessing.reductions import reduce_tensor

        world, rank = dist.get_world_size(group), dist.get_rank(group)
        gathered = torch.zeros((2, world, 3, int(m_cap)), dtype=torch.float32, device=device)
        signal = torch.zeros((world,), dtype=torch.int32, device=device)
        torch.cuda.synchronize(device)
        handles = [None] * world
        dist.all_gather_object(handles, (reduce_tensor(gathered), reduce_tensor(signal)), group=group)
        keep, pg, ps = [], [], []
        for r, (hg, hs) in enumerate(handles):
            g, sg = (gathered, signal) if r == rank else (hg[0](*hg[1]), hs[0](*hs[1]))
            keep += [g, sg]
            pg.append(g.data_ptr())
            ps.append(sg.data_ptr())
        self = cls.from_buffers(gathered, signal, pg, ps, rank, world)
        self._mapped = keep  # the peers' mappings live as long as the exchange
        dist.barrier(group)
        return self

    @classmethod
    def from_buffers(cls, gathered: torch.Tensor, signal: torch.Tensor, peer_gathered: list, peer_signal: list,
                     rank: int, world: int) -> "P2PExchange":
        """Peers given as raw device pointers (e.g. CUDA-IPC mappings of the
        other processes' [2, P, 3, m] gathered blocks); ``signal`` must be
        zeroed on every rank before the first push."""
        self = cls.__new__(cls)
        self._init(gathered, signal, peer_gathered, peer_signal, rank, world)
        return self

    def _init(self, gathered, signal, peer_gathered, peer_signal, rank, world):
        if gathered.dim() != 4 or gathered.shape[0] != 2 or gathered.shape[1] != world or gathered.shape[2] != 3:
            raise ValueError("gathered must be [2, world, 3, m_cap] fp32 (double-buffered by epoch parity)")
        device = gathered.device
        self.world, self.rank, self.m_cap = int(world), int(rank), int(gathered.shape[-1])
        self.gathered, self.signal = gathered, signal
        self._peer_gathered = torch.tensor([int(p) for p in peer_gathered], dtype=torch.int64, device=device)
        self._peer_signal = torch.tensor([int(p) for p in peer_signal], dtype=torch.int64, device=device)
        self._done = torch.zeros(1, dtype=torch.int32, device=device)
        self.epoch = 0

    @property
    def current(self) -> torch.Tensor:
        """[P, 3, m] half of ``gathered`` written by the latest push."""
        return self.gathered[self.epoch & 1]

    def push(self, part_max, part_sum, part_arg, S: int, stride: int, m_dev=None, m_host: int = 0, stream=None):
        import ctypes

        from . import _native
        from .hotpath import _p, _s

        self.epoch = (self.epoch + 1) & 0xFFFFFFFF or 1
        _native.call("mosaic_stats_exchange_push", _p(part_max), _p(part_sum), _p(part_arg), int(S), int(stride),
                     _p(m_dev), int(m_host), self.m_cap, _p(self._peer_gathered), _p(self._peer_signal),
                     self.rank, self.world, ctypes.c_uint32(self.epoch), _p(self._done), _s(stream))

    def wait(self, stream=None):
        import ctypes

        from . import _native
        from .hotpath import _p, _s

        _native.call("mosaic_stats_exchange_wait", _p(self.signal), self.world, ctypes.c_uint32(self.epoch),
                     _s(stream))


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
