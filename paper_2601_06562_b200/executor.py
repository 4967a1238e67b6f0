"""Numeric step executor: runs an instantiated step graph on the B200 with every
activation at its planned offset inside one cuMem arena.

The reference plans a denoising step but never executes it (the step loop
mosaic/workload.py:349-399 stops at the memory trace). Here
``StepExecutor.run`` walks ``ConcreteGraph.ops`` in order and dispatches on
``OpInstance.kind``; each tensor instance is a zero-copy view of the arena at
the offset ``plan_first_fit`` gave its storage group, so in-place pairs share
storage, chunk instances live exactly where the plan put them, and the step
allocates nothing per op. Graph inputs (token ids, mask indices, weights)
live outside the workspace, as in the reference (mosaic/liveness.py:52-53).

Op kinds (mosaic/workload.py:179-316, plus the fused-logits kinds):

* embed / matmul / fused_attention (K11 rotary positions + PyTorch SDPA) /
  add / alloc — model forward (not the hot path);
* ffn_up / ffn_gate / glu (K6) / activation / ffn_down / chunk_write — the
  lazily chunked FFN, rows [i*ceil(L/K_FFN), ...) per iteration; with
  ``fused_ffn``: ffn_gate_up (K10 + SwiGLU epilogue) / ffn_down_res (K10 +
  residual epilogue: down, chunk_write and the residual add in one launch);
* gather (K2) / lmhead_stats (K3) / sample (K4) / commit (K5) — the fused
  mask-only logits + remask hot path (``logits_mode="fused"``); in runs mode
  (default) the gather compacts only the rows of K3 tiles that are not one
  contiguous run of h, and K3 reads the run tiles from h by TMA;
* gather_logits / logits / shift / chunk_write / sample — the reference's
  materialising modes (``mask_only`` / ``eager``), executed with cuBLAS and
  fp32 softmax as the dense-logits baseline.
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Optional

import torch
import torch.nn.functional as F

from . import hotpath
from .errors import InputError
from .graph import ConcreteGraph, InstKey
from .liveness import LifetimeTable, analyze
from .planner import MemoryPlan, plan_first_fit
from .vmm import Workspace
from .workload import ModelConfig

_INT32_TENSORS = {"token_out", "token_ids", "mask_idx", "route_row", "route_pos", "expert_off"}
ATTN_BLOCK = 32768  # query rows per attention call


class RandomDLLM:
    """Random-init weights of a :class:`ModelConfig` on one device (bf16), in the
    template's graph-input layout. The LM head is stored [V, d] (K-major for
    K3); the reference's [d, V] is the same matrix transposed.

    ``distinct_layers`` limits how many layer weight sets are materialised;
    layer i uses set ``i % distinct_layers`` (the context sweep allocates all
    of them to charge the full weight footprint). ``rope_theta`` (LLaDA-8B's
    500000 by default; None = no positions) sets the rotary embedding K11
    applies to q and k inside ``fused_attention``."""

    def __init__(self, cfg: ModelConfig, device, seed: int = 0, distinct_layers: Optional[int] = None,
                 vocab_shard: tuple[int, int] | None = None, rope_theta: Optional[float] = 500000.0):
        if cfg.moe is not None and cfg.logits_mode not in ("fused", "fused_gather"):
            raise InputError("MoE models execute through the fused template (logits_mode='fused'), "
                             "whose FFN block carries the expert routing")
        if cfg.element_size != 2:
            raise InputError("the executor runs bf16 models (element_size=2)")
        self.cfg = cfg
        g = torch.Generator(device=device).manual_seed(seed)
        d, f, V = cfg.d_model, cfg.d_ff, cfg.vocab_size
        out_scale = 1.0 / math.sqrt(2 * cfg.n_layers)

        def w(*shape, scale=0.02):
            return (torch.randn(shape, generator=g, device=device, dtype=torch.float32) * scale).to(torch.bfloat16)

        self.w_embed = w(V, d, scale=1.0)
        n_sets = cfg.n_layers if distinct_layers is None else max(1, min(distinct_layers, cfg.n_layers))
        self.layers = []
        E = cfg.moe.n_experts if cfg.moe else None
        fused = cfg.logits_mode in ("fused", "fused_gather")
        for _ in range(n_sets):
            lw = {"w_qkv": w(d, 3 * d), "w_attn_out": w(d, d, scale=0.02 * out_scale)}
            if E is not None:
                # K10 operands: gate/up interleaved K-major [E*2f, d]; down K-major [E*d, f]
                lw["w_router"] = w(d, E, scale=1.0 / math.sqrt(d))
                lw["w_gate_up"] = hotpath.interleave_gate_up(w(E, d, f), w(E, d, f)).view(E * 2 * f, d)
                lw["w_down"] = w(E, f, d, scale=0.02 * out_scale).transpose(1, 2).contiguous().view(E * d, f)
            elif cfg.fused_ffn and fused:
                lw["w_gate_up"] = hotpath.interleave_gate_up(w(d, f), w(d, f))  # [2f, d]
                lw["w_down"] = w(f, d, scale=0.02 * out_scale).t().contiguous()  # [d, f] K-major for K10
            else:
                lw.update(w_up=w(d, f), w_down=w(f, d, scale=0.02 * out_scale))
                if cfg.gated_ffn:
                    lw["w_gate"] = w(d, f)
            self.layers.append(lw)
        v0, v1 = vocab_shard or (0, V)
        self.vocab_offset = v0
        w_vocab = w(V, d)  # the full head from the same stream, so a shard is a slice of the unsharded model
        self.w_vocab = w_vocab if (v0, v1) == (0, V) else w_vocab[v0:v1].contiguous()  # [V_shard, d]
        del w_vocab
        self.rope_theta = rope_theta
        self.inv_freq = (None if rope_theta is None
                         else hotpath.rope_inv_freq(d // cfg.n_heads, float(rope_theta), device))

    def layer(self, i: int) -> dict:
        return self.layers[i % len(self.layers)]

    def nbytes(self) -> int:
        n = self.w_embed.numel() + self.w_vocab.numel()
        for lw in self.layers:
            n += sum(t.numel() for t in lw.values())
        return 2 * n


_ALLOCATOR = None


def _scratch_allocator():
    """One pluggable allocator over csrc/pool.cu for the process (each executor's
    MemPool draws from the region it selects before its step)."""
    global _ALLOCATOR
    if _ALLOCATOR is None:
        from . import _native

        _native.load()
        _ALLOCATOR = torch.cuda.memory.CUDAPluggableAllocator(str(_native.LIB_PATH), "mosaic_pool_alloc",
                                                              "mosaic_pool_free")
    return _ALLOCATOR


def _rows(n_total: int, trips: int, it: Optional[int]) -> tuple[int, int]:
    if it is None:
        return 0, n_total
    per = -(-n_total // trips)
    r0 = min(it * per, n_total)
    return r0, min(r0 + per, n_total)


class StepExecutor:
    """Executes step graphs of one model inside one :class:`Workspace` (cuda)."""

    def __init__(self, model: RandomDLLM, workspace: Workspace, mask_id: int, exec_layers: Optional[int] = None,
                 group=None, die_aware: Optional[bool] = None):
        if workspace.backend != "cuda":
            raise InputError("the executor needs a cuda workspace")
        self.model = model
        self.cfg = model.cfg
        self.ws = workspace
        self.mask_id = int(mask_id)
        self.shift = self.cfg.shift_mode != "none"
        self.exec_layers = exec_layers  # execute only the first n layers (context sweep)
        # vocab-sharded LM head (model built with vocab_shard): the sample op merges
        # this rank's splits, all-gathers the per-row triples and merges in rank order
        self.group = group
        self.world = 1
        if group is not None:
            import torch.distributed as dist

            self.world = dist.get_world_size(group)
        dev = torch.device("cuda", workspace.device)
        self.device = dev
        self._side: dict[int, dict] = {}
        # the optional die split of K3's dynamic unit schedule (csrc/lmhead.cu),
        # decided as in MaskOnlyHead (hotpath.die_aware_default: off by default)
        self._die_aware = die_aware
        self._die_table = None
        self._die_tried = False
        self._sched = torch.zeros(4, dtype=torch.int32, device=dev)  # K3's dynamic unit schedule
        self._sched_ffn = torch.zeros(4, dtype=torch.int32, device=dev)  # K10's
        # fused logits: runs-mode A path (K3 reads contiguous-run tiles of h by TMA, the gather op
        # compacts only the other tiles' rows); MOSAIC_A_RUNS=0 gathers every row
        self.a_runs = os.environ.get("MOSAIC_A_RUNS", "1") != "0"
        self._runs_src = None
        # torch-side step temporaries (attention outputs, cuBLAS scratch) live in a
        # region at the start of the arena, served by csrc/pool.cu through a MemPool;
        # the planned activations follow it (offsets shifted by its size)
        self.scratch_bytes = 0
        self._pool = None
        self._fitted_L = None
        # cuBLAS / cuBLASLt keep one workspace per handle and stream for the life of
        # the process: create it now, outside the step, so it is not charged to (and
        # pinned inside) the step's scratch region
        a = torch.zeros(64, 64, dtype=torch.bfloat16, device=dev)
        torch.matmul(a, a)
        torch.mm(a, a, out_dtype=torch.float32)
        if hotpath.die_aware_default(die_aware, 1 << 30, model.w_vocab.shape[0]):
            # measured now (a one-off probe with ~250 MB of scratch), not mid-step next to a full arena
            self._die_table = hotpath.die_table_or_none(dev)
            self._die_tried = True

    def _die(self, m_cap: int):
        if not hotpath.die_aware_default(self._die_aware, m_cap, self.model.w_vocab.shape[0]):
            return None
        if not self._die_tried:  # one probe per executor; None = the default schedule
            self._die_table = hotpath.die_table_or_none(self.device)
            self._die_tried = True
        return self._die_table

    # ---------------------------------------------------------------- scratch
    def scratch_bytes_for(self, L: int) -> int:
        """Size of the arena's torch-scratch region for a first step at length
        L: an upper bound on the attention call's temporaries for one query
        block (output [rows, d] bf16 + per-head log-sum-exp fp32, each rounded
        to the caching allocator's 2 MiB segments, doubled for staging) with
        32 MiB of headroom (measured use: one output block + 2 MiB). After the step the region is cut to its
        measured high-water mark (``_fit_scratch``); an undersized region fails
        loudly with torch's out-of-memory error."""
        cfg = self.cfg
        qb = min(L, ATTN_BLOCK)
        mib2 = 2 << 20
        blk = -(-(qb * cfg.d_model * 2) // mib2) * mib2
        lse = -(-(cfg.n_heads * qb * 4) // mib2) * mib2
        need = 2 * blk + 2 * lse + (32 << 20)
        return -(-need // self.ws.page_size) * self.ws.page_size

    def _ensure_scratch(self, need: int) -> None:
        from . import _native

        if need > self.scratch_bytes:  # create, or grow in place (live blocks stay where they are)
            if self.ws.committed_bytes < need:
                self.ws.commit_to(need)
            _native.call("mosaic_pool_bind", self.ws.device, ctypes.c_void_p(self.ws.base), int(need))
            self.scratch_bytes = need
        if self._pool is None:
            self._pool = torch.cuda.MemPool(_scratch_allocator().allocator())
            self.ws.on_close(self.close)

    def _fit_scratch(self) -> None:
        """Shrink the scratch region to what the step actually used (the
        caching allocator keeps those segments and reuses them every step)
        plus 8 MiB, so the arena's commitment is plan + measured scratch."""
        from . import _native

        used = self.pool_stats()["high_water"]
        want = -(-(used + (8 << 20)) // self.ws.page_size) * self.ws.page_size
        if used and want < self.scratch_bytes:
            _native.call("mosaic_pool_bind", self.ws.device, ctypes.c_void_p(self.ws.base), int(want))
            self.scratch_bytes = want

    def close(self) -> None:
        """Release the scratch pool before the arena goes away (called by the
        workspace's close): cached segments are returned, the region forgotten."""
        from . import _native

        if self._pool is None:
            return
        torch.cuda.synchronize(self.device)
        self._pool = None
        import gc

        gc.collect()
        torch.cuda.empty_cache()
        if self.ws.base is not None:
            live = self.pool_stats()["in_use"]
            if live:  # a library kept a block of the step's scratch past the step: it dangles once unmapped
                import warnings

                warnings.warn(f"{live} bytes of the arena's torch-scratch region are still held at close")
            _native.call("mosaic_pool_unbind", self.ws.device, ctypes.c_void_p(self.ws.base))
        self.scratch_bytes = 0
        self._fitted_L = None

    def pool_stats(self) -> dict:
        from . import _native

        vals = [ctypes.c_uint64() for _ in range(4)]
        _native.call("mosaic_pool_stats", self.ws.device, ctypes.c_void_p(self.ws.base),
                     *(ctypes.byref(v) for v in vals))
        return dict(zip(("in_use", "high_water", "allocs", "refused"), (int(v.value) for v in vals)))

    # ---------------------------------------------------------------- buffers
    def _side_buffers(self, L: int) -> dict:
        """Graph inputs outside the workspace: mask indices, their count and the
        K1/K5 scratch (mosaic/liveness.py:52-53 excludes graph inputs)."""
        if L not in self._side:
            self._side = {L: {
                # zero-filled once: every entry is always a valid position, so a
                # count below the graph's M can never send K2 out of bounds
                "mask_idx": torch.zeros(L, dtype=torch.int32, device=self.device),
                "m_dev": torch.zeros(1, dtype=torch.int32, device=self.device),
                "compact": torch.empty(hotpath.mask_compact_scratch_bytes(L), dtype=torch.uint8, device=self.device),
                "remask": torch.empty(hotpath.remask_scratch_bytes(), dtype=torch.uint8, device=self.device),
            }}
            if self.cfg.moe is not None:  # K8 per-CTA expert histogram (graph-input-like scratch)
                self._side[L]["route"] = torch.empty(
                    hotpath.moe_route_scratch_bytes(L, self.cfg.moe.n_experts), dtype=torch.uint8, device=self.device)
        return self._side[L]

    def _views(self, g: ConcreteGraph, table: LifetimeTable, plan: MemoryPlan) -> dict[InstKey, torch.Tensor]:
        offset = plan.offsets()
        views: dict[InstKey, torch.Tensor] = {}
        t = g.template
        for grp in table.groups:
            base = offset[grp.id]
            for key in grp.members:
                tid = key[0]
                shape = t.instance_shape(tid, g.bindings)
                es = t.tensor(tid).element_size
                if es == 2:
                    dtype = torch.bfloat16
                elif tid.rsplit(".", 1)[-1] in _INT32_TENSORS:
                    dtype = torch.int32
                else:
                    dtype = torch.float32
                if 0 in shape:
                    views[key] = torch.empty(shape, dtype=dtype, device=self.device)
                else:
                    views[key] = self.ws.view(self.scratch_bytes + base, shape, dtype)
        return views

    # ---------------------------------------------------------------- run
    def plan(self, g: ConcreteGraph) -> tuple[LifetimeTable, MemoryPlan]:
        table = analyze(g)
        return table, plan_first_fit(table)

    def run(self, g: ConcreteGraph, x: torch.Tensor, k_unmask: int,
            table: Optional[LifetimeTable] = None, plan: Optional[MemoryPlan] = None,
            keep: tuple[str, ...] = (), profile: bool = False) -> dict:
        """Execute one step; ``x`` (int32 [L] on device) is updated in place.
        Returns timing/memory measurements and the instances named in ``keep``
        (copied out of the arena before they can be overwritten). With
        ``profile`` every op is bracketed by CUDA events on the current stream
        and the result carries device milliseconds per op kind."""
        if table is None or plan is None:
            table, plan = self.plan(g)
        b = g.bindings
        L, M = b["L"], b["M"]
        if x.dtype != torch.int32 or x.numel() != L:
            raise InputError("x must be int32 [L]")
        kinds = {op.kind for op in g.ops}  # the graph, not the model config, fixes the logits mode
        fused = "lmhead_stats" in kinds or "lmhead_stats_gather" in kinds
        self._mode = "fused" if fused else ("mask_only" if "gather_logits" in kinds else "eager")
        # the B200 path runs the whole step in the arena: torch-side temporaries in the
        # scratch region (MemPool), activations at their planned offsets after it. The
        # reference's materialising modes are the dense-logits baselines: torch allocator.
        if fused and not (self._pool is not None and self._fitted_L == L):
            self._ensure_scratch(self.scratch_bytes_for(L))
        if self.scratch_bytes + plan.workspace_size > self.ws.committed_bytes:
            self.ws.commit_to(self.scratch_bytes + plan.workspace_size)
        side = self._side_buffers(L)
        views = self._views(g, table, plan)
        kept: dict[str, torch.Tensor] = {}
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        # K1: masked positions (graph input mask_idx) of the current sequence
        hotpath.mask_compact(x, self.mask_id, side["mask_idx"], side["m_dev"], side["compact"])
        mask_idx = side["mask_idx"][:M]
        skip_layers = set()
        if self.exec_layers is not None:
            skip_layers = {f"l{i}." for i in range(self.exec_layers, self.cfg.n_layers)}
        marks = []
        keep_dst = {key: torch.empty_like(views[key]) for op in g.ops for key in op.outputs if key[0] in keep}
        if "token_out" in keep:
            keep_dst.update({(n, None): torch.empty_like(views[(n, None)]) for n in ("token_out", "confidence")})
        from contextlib import nullcontext

        if fused:
            from . import _native

            _native.call("mosaic_pool_select", self.ws.device, ctypes.c_void_p(self.ws.base))
        with torch.cuda.use_mem_pool(self._pool) if fused else nullcontext():
            self._run_ops(g, views, x, mask_idx, side, k_unmask, skip_layers, profile, marks, keep_dst, kept)
        end.record()
        end.synchronize()
        peak_committed = self.ws.committed_bytes  # what this step ran with
        if fused and self._fitted_L != L:  # first step at this length: cut the scratch region to
            self._fit_scratch()             # its measured use and give the arena's tail back
            self._fitted_L = L
            self.ws.commit_to(self.scratch_bytes + plan.workspace_size)
        m_seen = int(side["m_dev"].item())  # K1's count; the step was planned for the binding M
        if m_seen != M:
            raise InputError(f"x holds {m_seen} masked positions but the step graph was instantiated for M={M} "
                             "(only the first min(count, M) masked rows were eligible for the commit)")
        by_kind: dict[str, float] = {}
        for kind, e0, e1 in marks:
            by_kind[kind] = by_kind.get(kind, 0.0) + e0.elapsed_time(e1)
        return {"ms": start.elapsed_time(end), "workspace_bytes": plan.workspace_size,
                "committed_bytes": self.ws.committed_bytes, "step_committed_bytes": peak_committed,
                "scratch_bytes": self.scratch_bytes,
                "pool": self.pool_stats() if fused else None, "ops": len(g.ops), "kept": kept,
                "ms_by_kind": by_kind}

    def _run_ops(self, g, views, x, mask_idx, side, k_unmask, skip_layers, profile, marks, keep_dst, kept) -> None:
        keep = {key[0] for key in keep_dst}
        for op in g.ops:
            if skip_layers and op.op_id[:op.op_id.find(".") + 1] in skip_layers:
                continue
            if profile:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record()
            self._dispatch(op, g, views, x, mask_idx, side, k_unmask)
            if profile:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record()
                marks.append((op.kind, e0, e1))
            # copies out of the arena (tests / profiling) into buffers allocated before the step
            for key in op.outputs:
                if key[0] in keep:
                    kept[key[0] if key[1] is None else f"{key[0]}@{key[1]}"] = keep_dst[key].copy_(views[key])
            if op.kind == "sample" and "token_out" in keep:
                for name in ("token_out", "confidence"):
                    kept[name] = keep_dst[(name, None)].copy_(views[(name, None)])

    # ---------------------------------------------------------------- ops
    def _dispatch(self, op, g: ConcreteGraph, v, x, mask_idx, side, k_unmask: int) -> None:
        kind = op.kind
        b = g.bindings
        L, M = b["L"], b["M"]
        cfg = self.cfg
        d = cfg.d_model
        if kind == "embed":
            torch.index_select(self.model.w_embed, 0, x, out=v[op.outputs[0]])
        elif kind == "matmul":
            self._matmul(op, v)
        elif kind == "fused_attention":
            q, k, vv = (v[key] for key in op.inputs)
            H = cfg.n_heads
            dh = d // H
            if self.model.inv_freq is not None:  # K11: positions, in place on q and k (read only here)
                hotpath.rope_qk_(q, k, H, self.model.inv_freq)
            qh, kh, vh = (t.view(L, H, dh).transpose(0, 1).unsqueeze(0) for t in (q, k, vv))
            out = v[op.outputs[0]].view(L, H, dh)
            # bidirectional dLLM attention, query-blocked so the library's output
            # temporary stays bounded ([ATTN_BLOCK, d]) at million-token contexts
            for q0 in range(0, L, ATTN_BLOCK):
                q1 = min(q0 + ATTN_BLOCK, L)
                # one expression: the block's output temporary is freed before the next block's
                out[q0:q1].copy_(F.scaled_dot_product_attention(qh[:, :, q0:q1], kh, vh, is_causal=False)
                                 .squeeze(0).transpose(0, 1))
        elif kind == "add":
            a, c = (v[key] for key in op.inputs)
            torch.add(a, c, out=v[op.outputs[0]])
        elif kind == "alloc":
            out = v[op.outputs[0]]
            if op.outputs[0][0].endswith("ffn_acc"):
                out.zero_()
        elif kind.startswith("moe_") or (self.cfg.moe is not None and kind in ("ffn_gate_up", "ffn_down")):
            self._moe(op, g, v, side)
        elif kind == "ffn_gate_up":  # K10: gate/up GEMM + SwiGLU epilogue -> act
            r0, r1 = _rows(L, b["K_FFN"], op.iteration)
            f = cfg.d_ff
            hotpath.ffn_gemm(v[op.inputs[0]][r0:r1], self._layer(op.op_id)["w_gate_up"], v[op.outputs[0]][: r1 - r0],
                             2 * f, m_host=r1 - r0, swiglu=True, sched=self._sched_ffn)
        elif kind == "ffn_down_res":  # K10: h_attn[rows] += act @ w_down (down + chunk_write + residual)
            r0, r1 = _rows(L, b["K_FFN"], op.iteration)
            if r1 > r0:
                act, h = v[op.inputs[0]], v[op.inputs[2]]
                hotpath.ffn_gemm(act[: r1 - r0], self._layer(op.op_id)["w_down"], h[r0:r1], d, m_host=r1 - r0,
                                 residual=True, sched=self._sched_ffn)
        elif kind == "identity":
            pass  # in-place output naming the mutated storage (planned as one storage group)
        elif kind in ("ffn_up", "ffn_gate"):
            layer = self._layer(op.op_id)
            r0, r1 = _rows(L, b["K_FFN"], op.iteration)
            w = layer["w_up" if kind == "ffn_up" else "w_gate"]
            torch.matmul(v[op.inputs[0]][r0:r1], w, out=v[op.outputs[0]][: r1 - r0])
        elif kind == "glu":
            r0, r1 = _rows(L, b["K_FFN"], op.iteration)
            n = (r1 - r0) * (cfg.moe.top_k if cfg.moe else 1)
            up, gate = v[op.inputs[0]], v[op.inputs[1]]
            hotpath.swiglu_(gate[:n], up[:n])  # act shares storage with up (in place)
        elif kind == "activation":
            r0, r1 = _rows(L, b["K_FFN"], op.iteration)
            up = v[op.inputs[0]][: (r1 - r0) * (cfg.moe.top_k if cfg.moe else 1)]
            up.copy_(F.silu(up))
        elif kind == "ffn_down":
            layer = self._layer(op.op_id)
            r0, r1 = _rows(L, b["K_FFN"], op.iteration)
            torch.matmul(v[op.inputs[0]][: r1 - r0], layer["w_down"], out=v[op.outputs[0]][: r1 - r0])
        elif kind == "chunk_write":
            src, dst = op.inputs
            if src[0] == "logits":  # shift_mode=concat: logits chunk -> logits_all rows
                r0, r1 = _rows(M if self._mode == "mask_only" else L, b["K_logits"], op.iteration)
            else:
                r0, r1 = _rows(L, b["K_FFN"], op.iteration)
            v[dst][r0:r1].copy_(v[src][: r1 - r0])
        elif kind == "gather":  # K2, fused mode
            r0, r1 = _rows(M, b["K_logits"], op.iteration)
            if r1 > r0 and self.a_runs:
                hc = v[op.outputs[0]]
                hotpath.gather_rows_scattered(v[op.inputs[0]], mask_idx[r0:r1], hc, hc.shape[0], m_host=r1 - r0,
                                              shift=self.shift)
                self._runs_src = (v[op.inputs[0]], mask_idx[r0:r1])  # h stays live across the loop (barrier)
            elif r1 > r0:
                hotpath.gather_rows(v[op.inputs[0]], mask_idx[r0:r1], v[op.outputs[0]], m_host=r1 - r0,
                                    shift=self.shift)
        elif kind == "lmhead_stats":  # K3
            r0, r1 = _rows(M, b["K_logits"], op.iteration)
            hc, buf = v[op.inputs[0]], v[op.outputs[0]]
            cap = hc.shape[0]
            S, _ = hotpath.lmhead_plan(cap, self.model.w_vocab.shape[0], d, max_splits=buf.shape[1] // 3)
            if 3 * S > buf.shape[1]:
                raise InputError(f"K3 wants {S} splits but the template reserved {buf.shape[1] // 3}")
            flat = buf.view(-1)
            pm, ps = flat[: S * cap].view(S, cap), flat[S * cap: 2 * S * cap].view(S, cap)
            pa = flat[2 * S * cap: 3 * S * cap].view(torch.int32).view(S, cap)
            if r1 > r0 and self._runs_src is not None:
                h, idx = self._runs_src
                self._runs_src = None
                hotpath.lmhead_stats_runs(h, idx, hc, self.model.w_vocab, S, pm, ps, pa, cap, m_host=r1 - r0,
                                          shift=self.shift, v_offset=self.model.vocab_offset,
                                          die_of_sm=self._die(cap), sched=self._sched)
            elif r1 > r0:
                hotpath.lmhead_stats(hc, self.model.w_vocab, S, pm, ps, pa, m_host=r1 - r0,
                                     v_offset=self.model.vocab_offset, die_of_sm=self._die(cap),
                                     sched=self._sched)
            self._last_splits = S
        elif kind == "lmhead_stats_gather":  # K3 gather mode: A rows read from h at mask_idx
            r0, r1 = _rows(M, b["K_logits"], op.iteration)
            h, buf = v[op.inputs[0]], v[op.outputs[0]]
            cap = buf.shape[0]
            S, _ = hotpath.lmhead_plan(cap, self.model.w_vocab.shape[0], d, max_splits=buf.shape[1] // 3)
            if 3 * S > buf.shape[1]:
                raise InputError(f"K3 wants {S} splits but the template reserved {buf.shape[1] // 3}")
            flat = buf.view(-1)
            pm, ps = flat[: S * cap].view(S, cap), flat[S * cap: 2 * S * cap].view(S, cap)
            pa = flat[2 * S * cap: 3 * S * cap].view(torch.int32).view(S, cap)
            if r1 > r0:
                idx = side["mask_idx"][r0:r0 + cap]  # the chunk's positions (rows past r1 never stored)
                hotpath.lmhead_stats_gather(h, idx, self.model.w_vocab, S, pm, ps, pa, cap, m_host=r1 - r0,
                                            shift=self.shift, v_offset=self.model.vocab_offset,
                                            die_of_sm=self._die(cap), sched=self._sched)
            self._last_splits = S
        elif kind == "sample":
            self._sample(op, g, v)
        elif kind == "gather_logits":  # reference mask-only: materialised [rows, V]
            r0, r1 = _rows(M, b["K_logits"], op.iteration)
            rows = mask_idx[r0:r1].long()
            if self.shift:
                rows = (rows - 1).clamp_min(0)
            h = v[op.inputs[0]]
            torch.matmul(h.index_select(0, rows), self.model.w_vocab.t(), out=v[op.outputs[0]][: r1 - r0])
        elif kind == "logits":  # reference eager: all L rows
            r0, r1 = _rows(L, b["K_logits"], op.iteration)
            h = v[op.inputs[0]]
            src = h[r0:r1] if not self.shift else h.index_select(
                0, (torch.arange(r0, r1, device=h.device) - 1).clamp_min(0))
            torch.matmul(src, self.model.w_vocab.t(), out=v[op.outputs[0]][: r1 - r0])
        elif kind == "shift":
            pass  # the shift was applied as a row remap when the logits were produced
        elif kind == "commit":
            tok, conf = v[op.inputs[0]], v[op.inputs[1]]
            if self._mode == "eager":  # rows are all positions: pick the masked ones
                tok = tok.index_select(0, mask_idx.long())
                conf = conf.index_select(0, mask_idx.long())
            # the device count (capped at the planned M) bounds the commit, so rows
            # past K1's count never reach x even if x disagrees with the binding
            hotpath.remask_commit(conf[:M].contiguous(), mask_idx, tok[:M].contiguous(), k_unmask, x,
                                  side["remask"], M, m_dev=side["m_dev"])
        else:
            raise InputError(f"no executor for op kind {kind!r} ({op.label})")

    def _moe(self, op, g: ConcreteGraph, v, side) -> None:
        """The MoE FFN chunk (workload._moe_ffn_block): K8 routing, K2 dispatch
        gather, K10 grouped gate/up (+SwiGLU) and down GEMMs over the expert
        segments (offsets stay on the device), K9 combine."""
        cfg = self.cfg
        E, k = cfg.moe.n_experts, cfg.moe.top_k
        L = g.bindings["L"]
        r0, r1 = _rows(L, g.bindings["K_FFN"], op.iteration)
        n = r1 - r0
        kind = op.kind
        if n <= 0:
            if kind == "moe_route":
                v[op.outputs[3]].zero_()
            return
        lw = self._layer(op.op_id)
        if kind == "moe_router":
            h = v[op.inputs[0]]
            torch.mm(h[r0:r1], lw["w_router"], out_dtype=torch.float32, out=v[op.outputs[0]][:n])
        elif kind == "moe_route":
            rrow, rpos, rw, off = (v[key] for key in op.outputs)
            hotpath.moe_route(v[op.inputs[0]][:n], k, rrow, rpos, rw, off, side["route"], row_base=r0)
        elif kind == "moe_dispatch":
            h, rrow = (v[key] for key in op.inputs)
            hotpath.gather_rows(h, rrow, v[op.outputs[0]][: n * k], m_host=n * k)
        elif kind == "ffn_gate_up":  # K10 grouped over the expert segments, SwiGLU epilogue
            xin, off = v[op.inputs[0]], v[op.inputs[2]]
            hotpath.ffn_gemm(xin[: n * k], lw["w_gate_up"], v[op.outputs[0]][: n * k], 2 * cfg.d_ff,
                             group_off=off, groups=E, swiglu=True, sched=self._sched_ffn)
        elif kind == "ffn_down":  # K10 grouped, written over the dispatch rows (in place)
            act, off = v[op.inputs[0]], v[op.inputs[2]]
            hotpath.ffn_gemm(act[: n * k], lw["w_down"], v[op.outputs[0]][: n * k], cfg.d_model,
                             group_off=off, groups=E, sched=self._sched_ffn)
        elif kind == "moe_combine":
            src, rpos, rw, acc = (v[key] for key in op.inputs)
            hotpath.moe_combine(src[: n * k], rpos, rw, k, acc[r0:r1])
        else:
            raise InputError(f"no executor for op kind {kind!r} ({op.label})")

    def _layer(self, op_id: str) -> dict:
        return self.model.layer(int(op_id[1:op_id.index(".")]))

    def _matmul(self, op, v) -> None:
        name = op.op_id.split(".", 1)[1]
        lw = self._layer(op.op_id)
        d = self.cfg.d_model
        src = v[op.inputs[0]]
        if name in ("q_proj", "k_proj", "v_proj"):
            j = "qkv".index(name[0])
            w = lw["w_qkv"][:, j * d:(j + 1) * d]
        elif name == "attn_proj":
            w = lw["w_attn_out"]
        else:
            raise InputError(f"unsupported matmul {op.op_id}")  # materialised attention scores
        torch.matmul(src, w, out=v[op.outputs[0]])

    def _sample(self, op, g: ConcreteGraph, v) -> None:
        b = g.bindings
        cfg = self.cfg
        L, M = b["L"], b["M"]
        if self._mode == "fused":  # K4 over the K3 partial triples
            src = v[op.inputs[0]]
            r0, r1 = _rows(M, b["K_logits"], op.iteration)
            if r1 <= r0:
                return
            cap = src.shape[0]
            S = self._last_splits
            flat = src.view(-1)
            pm, ps = flat[: S * cap], flat[S * cap: 2 * S * cap]
            pa = flat[2 * S * cap: 3 * S * cap].view(torch.int32)
            tok, conf = v[op.inputs[1]], v[op.inputs[2]]
            if self.group is None:
                hotpath.stats_merge(pm, ps, pa, S, cap, cap, m_host=r1 - r0, token=tok[r0:r1], conf=conf[r0:r1])
                return
            from .shard import exchange_triples

            n = r1 - r0
            loc = torch.empty((3, n), dtype=torch.float32, device=self.device)
            hotpath.stats_merge(pm, ps, pa, S, cap, n, m_host=n, out_max=loc[0], out_sum=loc[1],
                                out_arg=loc[2].view(torch.int32))
            gat = exchange_triples(loc, group=self.group)  # [P, 3, n], rank-major
            hotpath.stats_merge(gat[0, 0], gat[0, 1], gat[0, 2].view(torch.int32), self.world, 3 * n, n, m_host=n,
                                token=tok[r0:r1], conf=conf[r0:r1])
            return
        # reference modes: fp32 softmax statistics of materialised bf16 logits
        if len(op.outputs) == 2:  # concat: sample over logits_all after the loop
            z = v[op.inputs[0]]
            tok, conf = v[op.outputs[0]], v[op.outputs[1]]
            r0, r1 = 0, z.shape[0]
        else:
            z, tok, conf = (v[key] for key in op.inputs)
            rows = M if self._mode == "mask_only" else L
            r0, r1 = _rows(rows, b["K_logits"], op.iteration)
            z = z[: r1 - r0]
        zf = z.float()
        mx, arg = zf.max(dim=1)
        lse = torch.logsumexp(zf, dim=1)
        tok[r0:r1] = arg.to(torch.int32) + self.model.vocab_offset
        conf[r0:r1] = torch.exp(mx - lse)
