"""Device-side hot path: torch-tensor wrappers over the C ABI and the fused
mask-only logits + remask step.

Each wrapper enqueues on the current torch CUDA stream (or an explicit one)
and takes caller-owned output buffers, so a whole denoising step can run out
of one preplanned workspace. Reference anchors:

* K1 ``mask_compact``   — mask_idx graph input, mosaic/workload.py:199-200
* K2 ``gather_rows``    — indirect row fetch, mosaic/kernel.py:77
* K3 ``lmhead_stats``   — gather_gemm, mosaic/kernel.py:62-86 (fused, no [M,V])
* K4 ``stats_merge``    — `sample` op, mosaic/workload.py:306-308
* K5 ``remask_commit``  — `commit` op, mosaic/workload.py:315
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import torch

from . import _native
from .errors import InputError, MosaicError

ALIGN = 256


def _p(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _s(stream: Optional[torch.cuda.Stream]):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _req(t: torch.Tensor, dtype: torch.dtype, name: str, ndim: int | None = None) -> None:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InputError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise InputError(f"{name} must be {dtype}, got {t.dtype}")
    if ndim is not None and t.dim() != ndim:
        raise InputError(f"{name} must be {ndim}-D, got shape {tuple(t.shape)}")
    if not t.is_contiguous():
        raise InputError(f"{name} must be contiguous")


def l2_persisting_limit(nbytes: int) -> int:
    """Reserve up to ``nbytes`` of L2 for persisting (evict_last) lines on the
    current device; returns the limit in force."""
    got = ctypes.c_int64()
    _native.call("mosaic_l2_persisting_limit", int(nbytes), ctypes.byref(got))
    return got.value


# ----------------------------------------------------------------- K1 / K2
def mask_compact_scratch_bytes(L: int) -> int:
    return int(_native.value("mosaic_mask_compact_scratch_bytes", L))


def mask_compact(x: torch.Tensor, mask_id: int, idx_out: torch.Tensor, m_out: torch.Tensor,
                 scratch: torch.Tensor, stream=None) -> None:
    _req(x, torch.int32, "x", 1)
    _req(idx_out, torch.int32, "idx_out", 1)
    _req(m_out, torch.int32, "m_out")
    if idx_out.numel() < x.numel():
        raise InputError("idx_out must hold L entries")
    if scratch.numel() * scratch.element_size() < mask_compact_scratch_bytes(x.numel()):
        raise InputError("compaction scratch too small")
    _native.call("mosaic_mask_compact", _p(x), x.numel(), int(mask_id), _p(idx_out), _p(m_out),
                 _p(scratch), _s(stream))


def gather_rows(hidden: torch.Tensor, idx: torch.Tensor, out: torch.Tensor, m_dev=None,
                m_host: int = 0, shift: bool = False, stream=None) -> None:
    if hidden.dtype != torch.bfloat16 or hidden.dim() != 2 or not hidden.is_cuda:
        raise InputError("hidden must be a 2-D bf16 CUDA tensor")
    if hidden.stride(1) != 1:
        raise InputError("hidden rows must be contiguous")
    _req(out, torch.bfloat16, "out", 2)
    _req(idx, torch.int32, "idx", 1)
    if out.shape[1] != hidden.shape[1]:
        raise InputError("row width mismatch")
    _native.call("mosaic_gather_rows", _p(hidden), hidden.shape[0], hidden.stride(0), hidden.shape[1],
                 _p(idx), _p(m_dev), int(m_host), out.shape[0], int(bool(shift)), _p(out), _s(stream))


# ----------------------------------------------------------------- K3
def lmhead_plan(m_cap: int, v_shard: int, d: int, max_splits: Optional[int] = None) -> tuple[int, int]:
    """(n_splits, tiles_per_split) for K3 (mosaic_lmhead_plan). With
    ``max_splits`` (e.g. a graph template's reserved partial width) the split
    is coarsened to at most that many splits, still tiling the vocab evenly."""
    s = ctypes.c_int32()
    t = ctypes.c_int32()
    _native.call("mosaic_lmhead_plan", m_cap, v_shard, d, ctypes.byref(s), ctypes.byref(t))
    S, tps = s.value, t.value
    if max_splits is not None and S > max_splits:
        n_tiles = -(-int(v_shard) // 256)
        tps = -(-n_tiles // int(max_splits))
        S = -(-n_tiles // tps)
    return S, tps


def lmhead_sample(hc: torch.Tensor, weight: torch.Tensor, n_splits: int, pos: torch.Tensor, temperature: float,
                  seed: int, part_max, part_sum, part_arg, part_y, part_x, m_dev=None, m_host: int = 0,
                  v_offset: int = 0, stream=None, die_of_sm: Optional[torch.Tensor] = None,
                  sched: Optional[torch.Tensor] = None) -> None:
    """K3's sampling variant (mosaic_lmhead_sample): per split and 128-column
    half the untempered (max, sum-exp) plus the Gumbel-max token over
    x + T * g(seed, pos, v); partials hold 2 * n_splits rows (merge S = 2 n_splits)."""
    _req(hc, torch.bfloat16, "hc", 2)
    _req(weight, torch.bfloat16, "weight", 2)
    _req(pos, torch.int32, "pos", 1)
    m_cap, d = hc.shape
    if weight.shape[1] != d or hc.stride(0) != d or weight.stride(0) != d:
        raise InputError("hc [m, d] and weight [V, d] must be contiguous with the same d")
    for t, dt, n in ((part_max, torch.float32, "part_max"), (part_sum, torch.float32, "part_sum"),
                     (part_arg, torch.int32, "part_arg"), (part_y, torch.float32, "part_y"),
                     (part_x, torch.float32, "part_x")):
        _req(t, dt, n)
        if t.numel() < 2 * n_splits * m_cap:
            raise InputError(f"{n} must hold 2*n_splits*m_cap entries (two column halves per split)")
    if (die_of_sm is not None or sched is not None) and (sched is None or sched.numel() * sched.element_size() < 16):
        raise InputError("the dynamic schedule needs a 16-byte sched scratch")
    _native.call("mosaic_lmhead_sample", _p(hc), m_cap, _p(m_dev), int(m_host), _p(weight), weight.shape[0], d,
                 int(v_offset), int(n_splits), _p(pos), ctypes.c_float(float(temperature)),
                 ctypes.c_uint32(int(seed) & 0xFFFFFFFF), _p(part_max), _p(part_sum), _p(part_arg), _p(part_y),
                 _p(part_x), _p(die_of_sm), _p(sched), _s(stream))


def sample_merge(part_max, part_sum, part_arg, part_y, part_x, S: int, stride: int, m_cap: int, token, conf,
                 lse=None, m_dev=None, m_host: int = 0, stream=None) -> None:
    """K4 of the sampling variant: token = noisy argmax, conf = untempered p(token)."""
    _native.call("mosaic_sample_merge", _p(part_max), _p(part_sum), _p(part_arg), _p(part_y), _p(part_x), int(S),
                 int(stride), _p(m_dev), int(m_host), int(m_cap), _p(token), _p(lse), _p(conf), _s(stream))


_DIE_MAPS: dict = {}


def die_map(device=None) -> tuple[torch.Tensor, dict]:
    """The measured SM -> L2-die map of ``device`` (cached per process): a
    device uint8 tensor [num SMs] for the optional die split of K3's dynamic
    schedule, plus counts."""
    if device is None or torch.device(device).index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    else:
        dev = torch.device("cuda", torch.device(device).index)
    if dev.index not in _DIE_MAPS:
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        scratch = torch.empty(int(_native.value("mosaic_die_map_scratch_bytes", n_sm)), dtype=torch.uint8, device=dev)
        host = (ctypes.c_uint8 * n_sm)()
        n0, amb = ctypes.c_int32(), ctypes.c_int32()
        with torch.cuda.device(dev):
            _native.call("mosaic_die_map", host, n_sm, _p(scratch), ctypes.byref(n0), ctypes.byref(amb), _s(None))
        table = torch.tensor(list(host), dtype=torch.uint8, device=dev)
        _DIE_MAPS[dev.index] = (table, {"n_sm": n_sm, "die0_sms": n0.value, "ambiguous": amb.value})
        del scratch  # ~2x L2 of probe scratch: back to torch's caching allocator for reuse
    return _DIE_MAPS[dev.index]


def die_table_or_none(device) -> Optional[torch.Tensor]:
    """The die map for K3's die split, or None (undivided dynamic schedule) if
    the probe cannot run here -- e.g. too little free memory for its ~2x-L2
    scratch. The schedule is an optimisation only; the result is the same."""
    try:
        return die_map(device)[0]
    except (MosaicError, RuntimeError) as exc:  # torch OOM is a RuntimeError subclass
        import sys

        print(f"mosaic_b200: die map probe unavailable ({exc}); K3 uses the default schedule", file=sys.stderr)
        return None


def die_aware_default(die_aware: Optional[bool] = None, m_cap: int = 0, v_shard: int = 0) -> bool:
    """Whether K3's dynamic schedule uses the SM -> die map (die-0 pairs claim
    units from the front, die-1 pairs from the back). An explicit argument or
    MOSAIC_DIE_AWARE=0/1 decides; the default is off: with units claimed
    dynamically the pairs already walk one contiguous window of m-groups, and
    the die split measured slightly slower with more DRAM traffic (LLaDA 32k
    steady 1.320-1.324 M vs 1.329-1.333 M masked tok/s, DRAM 7.3 vs 5.8 GB per
    launch; Dream 128k 30.1 vs 23.3 GB, profiles/r02i_k3_dynamic_schedule.txt).
    ``m_cap`` / ``v_shard`` are kept for callers that size the decision."""
    if die_aware is not None:
        return bool(die_aware)
    env = os.environ.get("MOSAIC_DIE_AWARE")
    if env in ("0", "1"):
        return env == "1"
    return False


def lmhead_stats(hc: torch.Tensor, weight: torch.Tensor, n_splits: int, part_max: torch.Tensor,
                 part_sum: torch.Tensor, part_arg: torch.Tensor, m_dev=None, m_host: int = 0,
                 v_offset: int = 0, stream=None, die_of_sm: Optional[torch.Tensor] = None,
                 sched: Optional[torch.Tensor] = None) -> None:
    _req(hc, torch.bfloat16, "hc", 2)
    _req(weight, torch.bfloat16, "weight", 2)
    m_cap, d = hc.shape
    if weight.shape[1] != d:
        raise InputError(f"weight is {tuple(weight.shape)}, expected [V, {d}]")
    for t, dt, n in ((part_max, torch.float32, "part_max"), (part_sum, torch.float32, "part_sum"),
                     (part_arg, torch.int32, "part_arg")):
        _req(t, dt, n)
        if t.numel() < n_splits * m_cap:
            raise InputError(f"{n} must hold n_splits*m_cap entries")
    if die_of_sm is not None or sched is not None:  # dynamic unit schedule (+ die map), csrc/lmhead.cu
        if sched is None or sched.numel() * sched.element_size() < 16:
            raise InputError("the dynamic schedule needs a 16-byte sched scratch")
        _native.call("mosaic_lmhead_stats_die", _p(hc), m_cap, _p(m_dev), int(m_host), _p(weight),
                     weight.shape[0], d, int(v_offset), int(n_splits), _p(part_max), _p(part_sum),
                     _p(part_arg), _p(die_of_sm), _p(sched), _s(stream))
        return
    _native.call("mosaic_lmhead_stats", _p(hc), m_cap, _p(m_dev), int(m_host), _p(weight),
                 weight.shape[0], d, int(v_offset), int(n_splits), _p(part_max), _p(part_sum),
                 _p(part_arg), _s(stream))


def lmhead_stats_gather(hidden: torch.Tensor, idx: torch.Tensor, weight: torch.Tensor, n_splits: int,
                        part_max: torch.Tensor, part_sum: torch.Tensor, part_arg: torch.Tensor, m_cap: int,
                        m_dev=None, m_host: int = 0, shift: bool = False, v_offset: int = 0, stream=None,
                        die_of_sm: Optional[torch.Tensor] = None, sched: Optional[torch.Tensor] = None,
                        repeats: bool = False) -> None:
    """K3 in gather mode: the A rows come straight from ``hidden`` [n, d] at
    the masked positions ``idx`` (cp.async loader warps), no compacted
    buffer; ``die_of_sm``/``sched`` select the dynamic schedule (and its die split) as in
    :func:`lmhead_stats`. ``repeats``: ``idx`` may repeat a row (not strictly
    ascending), so no tile may be taken for a contiguous run."""
    if hidden.dtype != torch.bfloat16 or hidden.dim() != 2 or hidden.stride(1) != 1 or not hidden.is_cuda:
        raise InputError("hidden must be a 2-D bf16 CUDA tensor with contiguous rows")
    _req(idx, torch.int32, "idx", 1)
    _req(weight, torch.bfloat16, "weight", 2)
    d = hidden.shape[1]
    if weight.shape[1] != d:
        raise InputError(f"weight is {tuple(weight.shape)}, expected [V, {d}]")
    if idx.numel() < (m_cap if m_dev is not None else min(int(m_host), m_cap)):
        raise InputError("idx must cover the masked rows (m_cap entries with a device count)")
    for t, dt, n in ((part_max, torch.float32, "part_max"), (part_sum, torch.float32, "part_sum"),
                     (part_arg, torch.int32, "part_arg")):
        _req(t, dt, n)
        if t.numel() < n_splits * m_cap:
            raise InputError(f"{n} must hold n_splits*m_cap entries")
    if die_of_sm is not None or sched is not None:
        if sched is None or sched.numel() * sched.element_size() < 16:
            raise InputError("the dynamic schedule needs a 16-byte sched scratch")
        _native.call("mosaic_lmhead_stats_gather_die", _p(hidden), hidden.shape[0], hidden.stride(0), _p(idx),
                     _shift_flags(shift, repeats), int(m_cap), _p(m_dev), int(m_host), _p(weight), weight.shape[0], d,
                     int(v_offset), int(n_splits), _p(part_max), _p(part_sum), _p(part_arg), _p(die_of_sm),
                     _p(sched), _s(stream))
        return
    _native.call("mosaic_lmhead_stats_gather", _p(hidden), hidden.shape[0], hidden.stride(0), _p(idx),
                 _shift_flags(shift, repeats), int(m_cap), _p(m_dev), int(m_host), _p(weight), weight.shape[0], d,
                 int(v_offset), int(n_splits), _p(part_max), _p(part_sum), _p(part_arg), _s(stream))


def _shift_flags(shift: bool, repeats: bool) -> int:
    """The gather/runs entry points' shift word: bit 0 Dream's token shift,
    bit 1 ``idx`` may repeat rows (no contiguous-run tiles)."""
    return int(bool(shift)) | (2 if repeats else 0)


def lmhead_tile_rows(m_cap: int) -> int:
    """Rows of one K3 tile at this capacity (256 on a CTA pair, 128 on one CTA):
    the unit runs mode classifies as contiguous or scattered."""
    c = lmhead_config(m_cap)
    return int(c["cta_group"]) * int(c["a_rows"])


def gather_rows_scattered(hidden: torch.Tensor, idx: torch.Tensor, hc: torch.Tensor, m_cap: int, m_dev=None,
                          m_host: int = 0, shift: bool = False, repeats: bool = False, stream=None) -> None:
    """K2 in runs mode: compact into ``hc`` only the rows of K3 tiles (of
    :func:`lmhead_tile_rows` rows at this ``m_cap``) whose source rows are not
    one contiguous run of ``hidden``."""
    if hidden.dtype != torch.bfloat16 or hidden.dim() != 2 or hidden.stride(1) != 1 or not hidden.is_cuda:
        raise InputError("hidden must be a 2-D bf16 CUDA tensor with contiguous rows")
    _req(idx, torch.int32, "idx", 1)
    _req(hc, torch.bfloat16, "hc", 2)
    if hc.shape[1] != hidden.shape[1] or hc.shape[0] < m_cap:
        raise InputError(f"hc {tuple(hc.shape)} does not hold {m_cap} rows of width {hidden.shape[1]}")
    _native.call("mosaic_gather_rows_scattered", _p(hidden), hidden.shape[0], hidden.stride(0), hidden.shape[1],
                 _p(idx), _p(m_dev), int(m_host), int(m_cap), _shift_flags(shift, repeats), lmhead_tile_rows(m_cap),
                 _p(hc), _s(stream))


def lmhead_stats_runs(hidden: torch.Tensor, idx: torch.Tensor, hc: torch.Tensor, weight: torch.Tensor,
                      n_splits: int, part_max: torch.Tensor, part_sum: torch.Tensor, part_arg: torch.Tensor,
                      m_cap: int, m_dev=None, m_host: int = 0, shift: bool = False, v_offset: int = 0, stream=None,
                      die_of_sm: Optional[torch.Tensor] = None, sched: Optional[torch.Tensor] = None,
                      repeats: bool = False) -> None:
    """K3 in runs mode (the product default): each tile's A box comes by TMA
    from ``hidden`` (its source rows are one contiguous run) or from ``hc``,
    where :func:`gather_rows_scattered` compacted the other tiles' rows (call
    it first). Outputs identical to gather_rows + lmhead_stats."""
    if hidden.dtype != torch.bfloat16 or hidden.dim() != 2 or hidden.stride(1) != 1 or not hidden.is_cuda:
        raise InputError("hidden must be a 2-D bf16 CUDA tensor with contiguous rows")
    _req(idx, torch.int32, "idx", 1)
    _req(hc, torch.bfloat16, "hc", 2)
    _req(weight, torch.bfloat16, "weight", 2)
    d = hidden.shape[1]
    if weight.shape[1] != d or hc.shape[1] != d or hc.shape[0] < m_cap:
        raise InputError(f"weight {tuple(weight.shape)} / hc {tuple(hc.shape)} do not match [*, {d}] x {m_cap}")
    if idx.numel() < (m_cap if m_dev is not None else min(int(m_host), m_cap)):
        raise InputError("idx must cover the masked rows (m_cap entries with a device count)")
    for t, dt, n in ((part_max, torch.float32, "part_max"), (part_sum, torch.float32, "part_sum"),
                     (part_arg, torch.int32, "part_arg")):
        _req(t, dt, n)
        if t.numel() < n_splits * m_cap:
            raise InputError(f"{n} must hold n_splits*m_cap entries")
    if (die_of_sm is not None or sched is not None) and (sched is None or sched.numel() * sched.element_size() < 16):
        raise InputError("the dynamic schedule needs a 16-byte sched scratch")
    _native.call("mosaic_lmhead_stats_runs", _p(hidden), hidden.shape[0], hidden.stride(0), _p(idx),
                 _shift_flags(shift, repeats), int(m_cap), _p(m_dev), int(m_host), _p(hc), _p(weight), weight.shape[0], d,
                 int(v_offset), int(n_splits), _p(part_max), _p(part_sum), _p(part_arg), _p(die_of_sm), _p(sched),
                 _s(stream))


def lmhead_logits(hc: torch.Tensor, weight: torch.Tensor, out: torch.Tensor, m_dev=None,
                  m_host: int = 0, stream=None) -> None:
    _req(hc, torch.bfloat16, "hc", 2)
    _req(weight, torch.bfloat16, "weight", 2)
    _req(out, torch.float32, "out", 2)
    if out.shape[0] < hc.shape[0] or out.shape[1] < weight.shape[0]:
        raise InputError("logits output too small")
    _native.call("mosaic_lmhead_logits", _p(hc), hc.shape[0], _p(m_dev), int(m_host), _p(weight),
                 weight.shape[0], hc.shape[1], _p(out), out.stride(0), _s(stream))


# ----------------------------------------------------------------- K4 / K5
def lmhead_logits_gather(hidden: torch.Tensor, idx: torch.Tensor, weight: torch.Tensor, out: torch.Tensor,
                         m_dev=None, m_host: int = 0, shift: bool = False, stream=None) -> None:
    """Materialised logits out[r] = hidden[src(idx[r])] @ weight.T (fp32), A rows
    gathered inside K3 (no [m, d] buffer): the drop-in gather_gemm's kernel."""
    _req(hidden, torch.bfloat16, "hidden", 2)
    _req(weight, torch.bfloat16, "weight", 2)
    _req(idx, torch.int32, "idx", 1)
    if out.dtype != torch.float32 or out.stride(1) != 1 or out.shape[1] < weight.shape[0]:
        raise InputError("out must be fp32 [m, >= V] with contiguous rows")
    m = min(idx.numel(), out.shape[0])
    _native.call("mosaic_lmhead_logits_gather", _p(hidden), hidden.shape[0], hidden.stride(0), _p(idx), int(shift),
                 m, _p(m_dev), int(m_host), _p(weight), weight.shape[0], weight.shape[1], _p(out), out.stride(0),
                 _s(stream))


def lmhead_config(m_cap: int, gather: bool = False) -> dict:
    """The K3 configuration a launch over m_cap rows uses (mosaic_lmhead_config)."""
    out = (ctypes.c_int64 * 8)()
    _native.call("mosaic_lmhead_config", int(m_cap), int(bool(gather)), out)
    keys = ("cta_group", "stages", "a_rows", "k_step", "w_rows", "tmem_cols", "smem_bytes", "threads")
    return dict(zip(keys, (int(v) for v in out)))


def stats_merge(in_max, in_sum, in_arg, S: int, stride: int, m_cap: int, m_dev=None, m_host: int = 0,
                out_max=None, out_sum=None, out_arg=None, token=None, lse=None, conf=None,
                stream=None) -> None:
    _native.call("mosaic_stats_merge", _p(in_max), _p(in_sum), _p(in_arg), int(S), int(stride),
                 _p(m_dev), int(m_host), int(m_cap), _p(out_max), _p(out_sum), _p(out_arg),
                 _p(token), _p(lse), _p(conf), _s(stream))


def remask_scratch_bytes() -> int:
    return int(_native.value("mosaic_remask_scratch_bytes"))


def remask_commit(conf, pos, token, k: int, x, scratch, m_cap: int, m_dev=None, m_host: int = 0,
                  selected=None, stream=None) -> None:
    _native.call("mosaic_remask_commit", _p(conf), _p(pos), _p(token), _p(m_dev), int(m_host),
                 int(m_cap), int(k), _p(x), _p(selected), _p(scratch), _s(stream))


def remask_commit_segmented(conf, pos, token, x, m_cap: int, seg_len: int, n_seg: int, k: int = 0,
                            k_per_seg: Optional[torch.Tensor] = None, m_dev=None, m_host: int = 0,
                            selected=None, stream=None) -> None:
    """K5 per segment (batched sequences / blocks): rows whose position lies in
    [b * seg_len, (b + 1) * seg_len) form segment b, which commits its own k_b
    most confident rows (``k_per_seg[b]``, device int32, or ``k`` for all)."""
    if k_per_seg is not None:
        _req(k_per_seg, torch.int32, "k_per_seg", 1)
        if k_per_seg.numel() < n_seg:
            raise InputError("k_per_seg must hold one count per segment")
    _native.call("mosaic_remask_commit_segmented", _p(conf), _p(pos), _p(token), _p(m_dev), int(m_host),
                 int(m_cap), int(seg_len), int(n_seg), _p(k_per_seg), int(k), _p(x), _p(selected), _s(stream))


# ----------------------------------------------------------------- K11
def rope_inv_freq(head_dim: int, theta: float, device) -> torch.Tensor:
    """theta^(-2i/head_dim), i < head_dim/2, fp32 -- the same expression as the
    torch reference (tests/torch_reference.py)."""
    return 1.0 / (theta ** (torch.arange(0, head_dim, 2, dtype=torch.float32, device=device) / head_dim))


def rope_qk_(q: torch.Tensor, k: torch.Tensor, n_heads: int, inv_freq: torch.Tensor, pos0: int = 0,
             stream=None) -> None:
    """In place: rotary embedding of q and k ([L, n_heads * head_dim] bf16 rows;
    the rows may be strided, e.g. the q and k column blocks of one fused qkv)."""
    for t, n in ((q, "q"), (k, "k")):
        if not t.is_cuda or t.dtype != torch.bfloat16 or t.dim() != 2:
            raise InputError(f"{n} must be a 2-D bf16 CUDA tensor")
    if q.shape != k.shape or q.stride() != k.stride() or q.stride(1) != 1:
        raise InputError("q and k must be [L, d] row-major views of the same shape and stride")
    _req(inv_freq, torch.float32, "inv_freq", 1)
    dh = q.shape[1] // n_heads
    if inv_freq.numel() != dh // 2:
        raise InputError(f"inv_freq must hold head_dim/2 = {dh // 2} entries")
    _native.call("mosaic_rope_qk", _p(q), _p(k), q.shape[0], int(n_heads), int(dh), q.stride(0), _p(inv_freq),
                 int(pos0), _s(stream))


# ----------------------------------------------------------------- K6
def swiglu_(gate: torch.Tensor, up: torch.Tensor, stream=None) -> torch.Tensor:
    """In place: up = silu(gate) * up (bf16), the chunked FFN's `glu` op."""
    _req(gate, torch.bfloat16, "gate")
    _req(up, torch.bfloat16, "up")
    if gate.numel() != up.numel():
        raise InputError("gate/up size mismatch")
    _native.call("mosaic_swiglu", _p(gate), _p(up), up.numel(), _s(stream))
    return up


# ----------------------------------------------------------------- K8 / K9 (MoE FFN)
def moe_route_scratch_bytes(rows: int, n_experts: int) -> int:
    return int(_native.value("mosaic_moe_route_scratch_bytes", rows, n_experts))


def moe_route(logits: torch.Tensor, top_k: int, disp_row: torch.Tensor, comb_pos: torch.Tensor,
              comb_w: torch.Tensor, expert_off: torch.Tensor, scratch: torch.Tensor, row_base: int = 0,
              disp_w: Optional[torch.Tensor] = None, stream=None) -> None:
    """Top-k routing of router logits [rows, E] (fp32) and the stable
    (expert, row, j) dispatch order; see include/mosaic_b200.h K8."""
    if logits.dtype != torch.float32 or logits.dim() != 2 or logits.stride(1) != 1 or not logits.is_cuda:
        raise InputError("router logits must be a 2-D fp32 CUDA tensor with contiguous rows")
    rows, E = logits.shape
    n = rows * int(top_k)
    for t, dt, name in ((disp_row, torch.int32, "disp_row"), (comb_pos, torch.int32, "comb_pos"),
                        (comb_w, torch.float32, "comb_w"), (expert_off, torch.int32, "expert_off")):
        _req(t, dt, name)
    if disp_row.numel() < n or comb_pos.numel() < n or comb_w.numel() < n or expert_off.numel() < E + 1:
        raise InputError("routing outputs too small")
    if scratch.numel() * scratch.element_size() < moe_route_scratch_bytes(rows, E):
        raise InputError("routing scratch too small")
    _native.call("mosaic_moe_route", _p(logits), logits.stride(0), rows, E, int(top_k), int(row_base),
                 _p(disp_row), _p(disp_w), _p(comb_pos), _p(comb_w), _p(expert_off), _p(scratch), _s(stream))


def moe_combine(src: torch.Tensor, comb_pos: torch.Tensor, comb_w: torch.Tensor, top_k: int,
                out: torch.Tensor, stream=None) -> None:
    """out[r] = sum_j comb_w[r, j] * src[comb_pos[r, j]] (bf16, fp32 math)."""
    if src.dtype != torch.bfloat16 or src.dim() != 2 or src.stride(1) != 1:
        raise InputError("src must be 2-D bf16 with contiguous rows")
    if out.dtype != torch.bfloat16 or out.dim() != 2 or out.stride(1) != 1 or out.shape[1] != src.shape[1]:
        raise InputError("out must be 2-D bf16 [rows, d] with contiguous rows")
    _req(comb_pos, torch.int32, "comb_pos")
    _req(comb_w, torch.float32, "comb_w")
    rows = out.shape[0]
    if comb_pos.numel() < rows * top_k or comb_w.numel() < rows * top_k:
        raise InputError("combine tables too small")
    _native.call("mosaic_moe_combine", _p(src), src.stride(0), _p(comb_pos), _p(comb_w), rows, int(top_k),
                 src.shape[1], _p(out), out.stride(0), _s(stream))


# ----------------------------------------------------------------- K10 (FFN GEMM)
def interleave_gate_up(w_gate: torch.Tensor, w_up: torch.Tensor) -> torch.Tensor:
    """[.., K, F] gate/up weights (torch layout) -> K10's SwiGLU operand
    [.., 2F, K]: K-major, 128-row gate and up blocks alternating."""
    *lead, K, F = w_gate.shape
    if F % 128:
        raise InputError(f"d_ff={F} must be a multiple of 128 for the fused SwiGLU GEMM")
    g = w_gate.transpose(-1, -2).reshape(*lead, F // 128, 128, K)
    u = w_up.transpose(-1, -2).reshape(*lead, F // 128, 128, K)
    return torch.stack((g, u), dim=-3).reshape(*lead, 2 * F, K).contiguous()


def ffn_gemm(a: torch.Tensor, w: torch.Tensor, out: torch.Tensor, n: int, group_off: Optional[torch.Tensor] = None,
             groups: int = 1, m_host: int = 0, swiglu: bool = False, residual: bool = False,
             stream=None, sched: Optional[torch.Tensor] = None) -> None:
    """K10: out[rows of group g] = a[rows of g] @ w[g].T (bf16, fp32 accumulate),
    w = [groups * n, K] K-major; with ``swiglu`` out = silu(gate) * up, n/2
    columns; with ``residual`` out += a @ w.T in place (one bf16 rounding).
    ``sched`` (16 device bytes): the dynamic tile schedule (as K3's)."""
    if swiglu and residual:
        raise InputError("swiglu and residual epilogues are exclusive")
    if a.dtype != torch.bfloat16 or a.dim() != 2 or a.stride(1) != 1 or not a.is_cuda:
        raise InputError("a must be 2-D bf16 with contiguous rows")
    if out.dtype != torch.bfloat16 or out.dim() != 2 or out.stride(1) != 1:
        raise InputError("out must be 2-D bf16 with contiguous rows")
    _req(w, torch.bfloat16, "w")
    K = a.shape[1]
    if w.numel() != groups * n * K:
        raise InputError(f"w must hold groups*n*K = {groups * n * K} elements")
    if out.shape[1] < (n // 2 if swiglu else n):
        raise InputError("out has too few columns")
    if group_off is not None:
        _req(group_off, torch.int32, "group_off")
        if group_off.numel() < groups + 1:
            raise InputError("group_off needs groups + 1 entries")
    elif groups != 1:
        raise InputError("several groups need device offsets")
    if sched is not None and sched.numel() * sched.element_size() < 16:
        raise InputError("the dynamic schedule needs a 16-byte sched scratch")
    _native.call("mosaic_ffn_gemm_sched", _p(a), min(a.shape[0], out.shape[0]), a.stride(0), _p(group_off),
                 int(groups), int(m_host), _p(w), int(n), K, 2 if residual else int(bool(swiglu)), _p(out),
                 out.stride(0), _p(sched), _s(stream))


# ----------------------------------------------------------------- buffers
class BufferLayout:
    """Bump layout of named buffers inside one device block (256 B aligned)."""

    def __init__(self) -> None:
        self.entries: dict[str, tuple[int, tuple[int, ...], torch.dtype]] = {}
        self.size = 0

    def add(self, name: str, shape: tuple[int, ...], dtype: torch.dtype) -> None:
        n = 1
        for s in shape:
            n *= s
        nbytes = n * torch.empty((), dtype=dtype).element_size()
        off = (self.size + ALIGN - 1) // ALIGN * ALIGN
        self.entries[name] = (off, tuple(shape), dtype)
        self.size = off + max(nbytes, 1)

    def views(self, block: torch.Tensor) -> dict[str, torch.Tensor]:
        if block.dtype != torch.uint8 or block.numel() < self.size:
            raise InputError("buffer block too small for the layout")
        out = {}
        for name, (off, shape, dtype) in self.entries.items():
            n = 1
            for s in shape:
                n *= s
            nbytes = n * torch.empty((), dtype=dtype).element_size()
            out[name] = block[off:off + nbytes].view(dtype).view(shape)
        return out


@dataclass
class StepOutput:
    m_dev: torch.Tensor       # [1] int32, masked rows this step
    idx: torch.Tensor         # [m_cap] int32 masked positions (ascending), first M valid
    token: torch.Tensor       # [m_cap] int32 argmax token per masked row
    lse: torch.Tensor         # [m_cap] fp32 log-sum-exp
    conf: torch.Tensor        # [m_cap] fp32 p(token)
    selected: torch.Tensor    # [m_cap] int32 1 = unmasked this step
    offset: int = 0           # positions are idx + offset (a windowed step's lo)


class MaskOnlyHead:
    """The fused mask-only logits + remask step on one vocab shard.

    step(x, hidden, k): compact the masked positions of ``x`` (K1), gather their
    hidden rows (K2), run the LM-head statistics GEMM over this rank's vocab
    shard (K3), merge the splits (K4), combine the per-row triples across the
    vocab-sharded ranks (all-gather over NCCL + K4 in rank order), and commit the
    k most confident predictions into ``x`` in place (K5). ``[M, V]`` logits
    never exist. Every rank of ``group`` ends with identical ``x``.

    ``m_cap`` (default ``seq_len``) sizes the per-row buffers; the masked count
    M is read on the device every step, so a step with more than ``m_cap``
    masked positions processes only the first ``m_cap`` of them (ascending
    positions) -- size it for the largest M the caller will present (the step-0
    count of the schedule, ``workload.ScenarioConfig.masked_at(0)``).
    """

    def __init__(self, weight_shard: torch.Tensor, *, seq_len: int, mask_id: int,
                 vocab_offset: int = 0, m_cap: Optional[int] = None, shift: bool = False,
                 group=None, block: Optional[torch.Tensor] = None, fused_gather: bool = False,
                 exchange="nccl", die_aware: Optional[bool] = None, temperature: float = 0.0, seed: int = 0):
        _req(weight_shard, torch.bfloat16, "weight_shard", 2)
        self.weight = weight_shard
        self.v_shard, self.d = weight_shard.shape
        self.vocab_offset = int(vocab_offset)
        self.L = int(seq_len)
        self.m_cap = int(m_cap if m_cap is not None else seq_len)
        self.mask_id = int(mask_id)
        self.shift = bool(shift)
        self.group = group
        self.fused_gather = bool(fused_gather)  # K3 reads rows of `hidden` directly: no K2, no hc buffer
        # otherwise runs mode: K3 reads contiguous-run tiles from `hidden`, K2 compacts only the other
        # tiles' rows into hc (MOSAIC_A_RUNS=0: every row through K2, the round-1 buffered path)
        self.a_runs = not self.fused_gather and temperature == 0 and os.environ.get("MOSAIC_A_RUNS", "1") != "0"
        # temperature > 0: Gumbel-max sampling in K3's epilogue (LLaDA generate's sampler), one fresh
        # noise draw per step from (seed, step counter); single-process, buffered A path
        self.temperature = float(temperature)
        self.seed = int(seed)
        self._steps = 0
        if self.temperature < 0:
            raise InputError("temperature must be >= 0")
        if self.temperature > 0 and (group is not None or hasattr(exchange, "push") or self.fused_gather):
            raise InputError("sampling (temperature > 0) runs on single-process heads with the buffered A path")
        self._die_aware = die_aware
        self._wplans: dict = {}
        self.die_table = (die_table_or_none(weight_shard.device)
                          if die_aware_default(die_aware, self.m_cap, self.v_shard) else None)
        if not (exchange in ("nccl", "p2p", "p2p_ipc") or hasattr(exchange, "push")):
            raise InputError(f"exchange must be 'nccl', 'p2p', 'p2p_ipc' or a P2PExchange, got {exchange!r}")
        self.exchange = exchange
        self.world = 1
        if group is not None:
            import torch.distributed as dist
            self.world = dist.get_world_size(group)
        self.n_splits, self.tiles_per_split = lmhead_plan(self.m_cap, self.v_shard, self.d)
        lay = BufferLayout()
        m, S, P = self.m_cap, self.n_splits, self.world
        lay.add("idx", (max(self.L, m),), torch.int32)
        lay.add("m_dev", (1,), torch.int32)
        lay.add("compact_scratch", (mask_compact_scratch_bytes(self.L),), torch.uint8)
        if not self.fused_gather:
            lay.add("hc", (m, self.d), torch.bfloat16)
        Sp = 2 * S if self.temperature > 0 else S  # the sampling variant writes two halves per split
        lay.add("part_max", (Sp, m), torch.float32)
        lay.add("part_sum", (Sp, m), torch.float32)
        lay.add("part_arg", (Sp, m), torch.int32)
        if self.temperature > 0:
            lay.add("part_y", (Sp, m), torch.float32)
            lay.add("part_x", (Sp, m), torch.float32)
        if group is not None:  # the exchange path runs whenever a process group is given (even P = 1)
            lay.add("local", (3, m), torch.float32)     # merged (max, sum, arg-bits) of this shard
            lay.add("gathered", (P, 3, m), torch.float32)
        lay.add("token", (m,), torch.int32)
        lay.add("lse", (m,), torch.float32)
        lay.add("conf", (m,), torch.float32)
        lay.add("selected", (m,), torch.int32)
        lay.add("remask_scratch", (remask_scratch_bytes(),), torch.uint8)
        lay.add("sched", (4,), torch.int32)
        self.layout = lay
        self.p2p = None
        if hasattr(exchange, "push"):  # a prepared P2PExchange (peer buffers set up by the caller)
            self.p2p = exchange
            self.world = exchange.world
        elif group is not None and exchange in ("p2p", "p2p_ipc"):
            from .shard import P2PExchange

            if exchange == "p2p":  # peers through torch symmetric memory (one GPU per rank)
                self.p2p = P2PExchange(self.m_cap, group, weight_shard.device)
            else:  # peers through CUDA IPC handles (ranks sharing a GPU)
                self.p2p = P2PExchange.ipc(self.m_cap, group, weight_shard.device)
        if block is None:
            block = torch.empty(lay.size, dtype=torch.uint8, device=weight_shard.device)
        self.block = block
        self.buf = lay.views(block)

    @property
    def workspace_bytes(self) -> int:
        return self.layout.size

    def step_batch(self, x: torch.Tensor, hidden: torch.Tensor, k, stream=None,
                   window: Optional[tuple[int, int]] = None) -> StepOutput:
        """One step over a batch of B sequences at once: ``x`` [B, Ls] int32,
        ``hidden`` [B, Ls, d] bf16 (contiguous), ``k`` an int or a device int32
        [B] of per-sequence unmask counts, ``window=(lo, hi)`` the same block of
        every sequence (semi-autoregressive decoding) or None for all of it.
        All B x (hi - lo) positions share one LM-head pass -- so a batch of short
        blocks streams W once instead of B times -- and every sequence commits
        its own k most confident masked positions (segmented K5). The head must
        be built with ``seq_len >= B * (hi - lo)``; the returned ``idx`` are the
        flattened window coordinates b * (hi - lo) + (p - lo)."""
        from contextlib import nullcontext

        if x.dim() != 2 or x.dtype != torch.int32 or not x.is_cuda:
            raise InputError("x must be a [B, Ls] int32 CUDA tensor")
        B, Ls = x.shape
        if hidden.shape != (B, Ls, self.d) or hidden.dtype != torch.bfloat16 or not hidden.is_contiguous():
            raise InputError(f"hidden must be a contiguous [{B}, {Ls}, {self.d}] bf16 tensor")
        lo, hi = (0, Ls) if window is None else (int(window[0]), int(window[1]))
        if not 0 <= lo < hi <= Ls:
            raise InputError(f"window {window} outside [0, {Ls})")
        Wn = hi - lo
        if B * Wn > self.L:
            raise InputError(f"batch x window = {B * Wn} positions exceeds the head's seq_len {self.L}")
        b = self.buf
        m = min(self.m_cap, B * Wn)
        S, die = self._window_plan(m)
        if getattr(self, "_xs", None) is None:  # batch staging (first batched call)
            self._xs = torch.empty(self.L, dtype=torch.int32, device=self.weight.device)
            self._rows = torch.empty(self.m_cap, dtype=torch.int32, device=self.weight.device)
        with torch.cuda.stream(stream) if stream is not None else nullcontext():
            xs = self._xs[:B * Wn].view(B, Wn)
            xs.copy_(x[:, lo:hi])
            mask_compact(xs.view(-1), self.mask_id, b["idx"], b["m_dev"], b["compact_scratch"], stream)
            q = b["idx"][:m]
            if window is None and not self.shift:
                rows = q  # flattened positions are the hidden rows
            else:  # q = seq * Wn + j -> hidden row seq * Ls + src(lo + j), src(p) = max(p - 1, 0) with the shift
                rows = self._rows[:m]
                _native.call("mosaic_window_rows", _p(q), _p(b["m_dev"]), 0, m, Wn, Ls, lo, int(self.shift),
                             _p(rows), _s(stream))
            # with the shift and lo = 0, src(0) = src(1): the rows repeat, so no tile is a contiguous run
            self._stats(hidden.view(B * Ls, self.d), rows, False, m, S, die, stream, keys=q,
                        repeats=self.shift and lo == 0)
            kt = k if isinstance(k, torch.Tensor) else None
            remask_commit_segmented(b["conf"], q, b["token"], xs.view(-1), m, Wn, B,
                                    k=0 if kt is not None else int(k), k_per_seg=kt, m_dev=b["m_dev"],
                                    selected=b["selected"], stream=stream)
            x[:, lo:hi].copy_(xs)
        return StepOutput(b["m_dev"], b["idx"][:m], b["token"], b["lse"], b["conf"], b["selected"], lo)

    def capture(self, x: torch.Tensor, hidden: torch.Tensor, k: int,
                window: Optional[tuple[int, int]] = None) -> "torch.cuda.CUDAGraph":
        """Capture one whole step (K1..K5) into a CUDA graph bound to these
        ``x`` / ``hidden`` buffers and this ``k`` (a [B, Ls] ``x`` captures
        :meth:`step_batch`). Every launch reads the masked
        count from the device (K1's output), so one graph serves every step of
        a run whatever M is: refill ``x`` / ``hidden`` in place and ``replay()``.
        Nothing runs during capture (``x`` is untouched until the first replay).
        Single-process heads only (the exchange paths are not captured)."""
        if self.group is not None or self.p2p is not None:
            raise InputError("graph capture is for single-process heads")
        if self.temperature > 0:
            raise InputError("a captured sampling step would replay the same noise every step: use step()")
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=x.device)
        side.wait_stream(torch.cuda.current_stream(x.device))
        batched = x.dim() == 2  # [B, Ls]: capture step_batch
        if batched:
            B, Ls = x.shape
            lo, hi = (0, Ls) if window is None else window
            self._window_plan(min(self.m_cap, B * (int(hi) - int(lo))))  # host planning before capture
            if getattr(self, "_xs", None) is None:  # staging buffers must exist before capture
                self._xs = torch.empty(self.L, dtype=torch.int32, device=self.weight.device)
                self._rows = torch.empty(self.m_cap, dtype=torch.int32, device=self.weight.device)
        elif window is not None:
            self._window_plan(min(self.m_cap, int(window[1]) - int(window[0])))  # host planning before capture
        with torch.cuda.graph(g, stream=side):
            if batched:
                self.step_batch(x, hidden, k, window=window)
            else:
                self.step(x, hidden, k, window=window)
        torch.cuda.current_stream(x.device).wait_stream(side)
        return g

    def _window_plan(self, m_w: int) -> tuple[int, Optional[torch.Tensor]]:
        """Splits and die table for a windowed step of capacity m_w rows: planned
        for m_w itself (a block of 32 masked rows wants one split per SM, not the
        full-sequence split), coarsened if needed to fit the head's partials."""
        if m_w not in self._wplans:
            S_w, _ = lmhead_plan(m_w, self.v_shard, self.d)
            if S_w * m_w > self.n_splits * self.m_cap:
                S_w, _ = lmhead_plan(m_w, self.v_shard, self.d,
                                     max_splits=max(1, self.n_splits * self.m_cap // m_w))
            die = self.die_table if die_aware_default(self._die_aware, m_w, self.v_shard) else None
            self._wplans[m_w] = (S_w, die)
        return self._wplans[m_w]

    def _stats(self, hidden: torch.Tensor, rows: torch.Tensor, shift: bool, m: int, S: int, die, stream,
               keys: Optional[torch.Tensor] = None, repeats: bool = False) -> None:
        """K2 + K3 (or gather-mode K3) over the hidden rows ``rows[r]`` (src(p)
        = p - 1 with ``shift``) of the M compacted rows, then K4 -- through the
        vocab-shard exchange when the head is sharded -- into token/lse/conf.
        ``keys[r]`` (default ``rows``) keys the sampling noise: the window
        coordinate of the row, never the hidden row it reads, so two positions
        sharing a hidden row (the shift at p = 0, 1) draw independent noise and
        ``step_batch`` with B = 1 draws what ``step`` draws."""
        b = self.buf
        pmax = b["part_max"].view(-1)[:S * m].view(S, m)
        psum = b["part_sum"].view(-1)[:S * m].view(S, m)
        parg = b["part_arg"].view(-1)[:S * m].view(S, m)
        m_dev = b["m_dev"]
        if self.fused_gather:
            lmhead_stats_gather(hidden, rows, self.weight, S, pmax, psum, parg, m, m_dev=m_dev, shift=shift,
                                v_offset=self.vocab_offset, stream=stream, die_of_sm=die, sched=b["sched"],
                                repeats=repeats)
        elif self.temperature > 0:  # Gumbel-max sampling in K3's epilogue, noise keyed by keys[r]
            hc = b["hc"][:m]
            gather_rows(hidden, rows, hc, m_dev=m_dev, shift=shift, stream=stream)
            S2 = 2 * S  # two 128-column halves per split
            pm2, ps2, pa2 = (b[n].view(-1)[:S2 * m].view(S2, m) for n in ("part_max", "part_sum", "part_arg"))
            py = b["part_y"].view(-1)[:S2 * m].view(S2, m)
            px = b["part_x"].view(-1)[:S2 * m].view(S2, m)
            seed = (self.seed * 0x9E3779B1 + self._steps * 0x85EBCA6B + 0x27D4EB2F) & 0xFFFFFFFF
            self._steps += 1
            lmhead_sample(hc, self.weight, S, rows if keys is None else keys, self.temperature, seed, pm2, ps2, pa2, py, px, m_dev=m_dev,
                          v_offset=self.vocab_offset, stream=stream, die_of_sm=die, sched=b["sched"])
            sample_merge(pm2, ps2, pa2, py, px, S2, m, m, b["token"], b["conf"], lse=b["lse"], m_dev=m_dev,
                         stream=stream)
            return
        elif self.a_runs:
            gather_rows_scattered(hidden, rows, b["hc"][:m], m, m_dev=m_dev, shift=shift, repeats=repeats,
                                  stream=stream)
            lmhead_stats_runs(hidden, rows, b["hc"][:m], self.weight, S, pmax, psum, parg, m, m_dev=m_dev,
                              shift=shift, v_offset=self.vocab_offset, stream=stream, die_of_sm=die,
                              sched=b["sched"], repeats=repeats)
        else:
            hc = b["hc"][:m]
            gather_rows(hidden, rows, hc, m_dev=m_dev, shift=shift, stream=stream)
            lmhead_stats(hc, self.weight, S, pmax, psum, parg, m_dev=m_dev, v_offset=self.vocab_offset,
                         stream=stream, die_of_sm=die, sched=b["sched"])
        if self.group is None and self.p2p is None:
            stats_merge(pmax, psum, parg, S, m, m, m_dev=m_dev, token=b["token"], lse=b["lse"], conf=b["conf"],
                        stream=stream)
        elif self.p2p is not None:  # K4x: merge + peer stores + signal, then wait; no NCCL call
            self.p2p.push(pmax, psum, parg, S, m, m_dev=m_dev, stream=stream)
            self.p2p.wait(stream)
            g = self.p2p.current
            M3 = 3 * self.p2p.m_cap
            stats_merge(g[0, 0], g[0, 1], g[0, 2].view(torch.int32), self.world, M3, m,
                        m_dev=m_dev, token=b["token"], lse=b["lse"], conf=b["conf"], stream=stream)
        else:
            from .shard import exchange_triples

            loc = b["local"]
            stats_merge(pmax, psum, parg, S, m, m, m_dev=m_dev,
                        out_max=loc[0], out_sum=loc[1], out_arg=loc[2].view(torch.int32),
                        stream=stream)
            g = b["gathered"]
            # NCCL orders its collective after torch's current stream: make that the step's stream
            with torch.cuda.stream(stream if stream is not None else torch.cuda.current_stream()):
                exchange_triples(loc, group=self.group, out=g)  # NCCL all-gather, 12 B/row/rank
            stats_merge(g[0, 0], g[0, 1], g[0, 2].view(torch.int32), self.world, 3 * self.m_cap, m,
                        m_dev=m_dev, token=b["token"], lse=b["lse"], conf=b["conf"], stream=stream)

    def step(self, x: torch.Tensor, hidden: torch.Tensor, k: int, stream=None,
             window: Optional[tuple[int, int]] = None) -> StepOutput:
        """One step. ``window=(lo, hi)``: only masked positions in [lo, hi) are
        predicted and only they can be committed (semi-autoregressive block
        decoding: the current block); everything runs on views of ``x`` /
        ``hidden``, so [M, V] work and buffers shrink to the window. The
        returned ``idx`` is then relative to ``lo`` (``StepOutput.offset``)."""
        b = self.buf
        _req(x, torch.int32, "x", 1)
        if x.numel() != self.L or hidden.shape[0] != self.L or hidden.shape[1] != self.d:
            raise InputError("x/hidden do not match the configured sequence length / width")
        lo, hi = (0, self.L) if window is None else (int(window[0]), int(window[1]))
        if not 0 <= lo < hi <= self.L:
            raise InputError(f"window {window} outside [0, {self.L})")
        shift = self.shift
        if (lo, hi) != (0, self.L):
            x = x[lo:hi]
            if shift and lo > 0:  # src(p) = p - 1 >= lo - 1: the shifted view needs no clamp
                hidden, shift = hidden[lo - 1:hi - 1], False
            else:
                hidden = hidden[lo:hi]
            m = min(self.m_cap, hi - lo)
            S, die = self._window_plan(m)
        else:
            m, S, die = self.m_cap, self.n_splits, self.die_table
        mask_compact(x, self.mask_id, b["idx"], b["m_dev"], b["compact_scratch"], stream)
        self._stats(hidden, b["idx"], shift, m, S, die, stream)
        remask_commit(b["conf"], b["idx"], b["token"], int(k), x, b["remask_scratch"], m,
                      m_dev=b["m_dev"], selected=b["selected"], stream=stream)
        return StepOutput(b["m_dev"], b["idx"][:m], b["token"], b["lse"], b["conf"], b["selected"], lo)
