"""Per-step planning at serving speed: instantiation + liveness skeletons cached
per chunk configuration and rebound to new sizes.

The reference re-instantiates, re-analyses and re-plans the whole step graph
at every denoising step (mosaic/workload.py:392-396 inside simulate_run, and
once per probe in the chunk search, mosaic/chunker.py:86-165). Only the trip
counts (K_logits, K_FFN) change the graph's *structure* -- the op instances,
their order, the storage groups and their live intervals; the sequence
length L and the masked count M (which shrinks every step) only change
tensor sizes. So the structure is built once per trip-count tuple and every
later step rebinds sizes in O(groups): a step's planning then costs the
rebind plus the native first-fit (csrc/planner.cu) instead of a full
instantiate + analyze in Python.

``instantiate_analyzed(template, bindings)`` returns exactly what
``analyze(template.instantiate(bindings))`` returns (tests/test_plancache.py
checks equality on every configuration the suites use).
"""
from __future__ import annotations

from collections import OrderedDict
from dataclasses import replace
from typing import Mapping

from .errors import InstantiationError
from .graph import ConcreteGraph, GraphTemplate, _volume
from .liveness import LifetimeTable, StorageGroup, analyze

_MAX_SKELETONS = 64


class _Skeleton:
    """Structure of one instantiation: graph ops, lifetime groups, and which
    template tensor sizes each storage group."""

    def __init__(self, template: GraphTemplate, g: ConcreteGraph, table: LifetimeTable):
        self.g = g
        self.table = table
        self.group_tid = [grp.members[0][0] for grp in table.groups]
        pairs = set()
        for op in g.ops:
            for out, src in op.in_place:
                pairs.add((out[0], src[0]))
        for a, b in g.aliases:
            pairs.add((a[0], b[0]))
        self.equal_pairs = tuple(sorted(pairs))
        self.keys = tuple(g.sizes)
        self.last_inst: dict[str, int] = {tid: g.sizes[grp.members[0]] for grp, tid in
                                          zip(table.groups, self.group_tid)}
        self.last_groups = list(table.groups)

    def rebind(self, template: GraphTemplate, bindings: dict) -> tuple[ConcreteGraph, LifetimeTable]:
        inst = {tid: template.tensors[tid].element_size * _volume(template._chunk_shape[tid], bindings)
                for tid in template.tensors}
        for out, src in self.equal_pairs:
            if inst[out] != inst[src]:
                raise InstantiationError(f"in_place/alias pair {out!r}<-{src!r} has mismatched sizes "
                                         f"{inst[out]} != {inst[src]} under {bindings}")
        sizes = {k: inst[k[0]] for k in self.keys}
        g = replace(self.g, bindings=dict(bindings), sizes=sizes)
        groups = self.last_groups
        for i, tid in enumerate(self.group_tid):
            if inst[tid] != groups[i].size:  # only the L/M-dependent groups change
                o = groups[i]
                groups[i] = StorageGroup(o.id, inst[tid], o.tag, o.def_index, o.last_use_index, o.members,
                                         o.chunkable_symbol)
        return g, LifetimeTable(groups=tuple(groups), length=self.table.length)


def _trip_key(template: GraphTemplate, bindings: Mapping[str, int]) -> tuple:
    template.freeze()
    return tuple((loop.trip_symbol, bindings[loop.trip_symbol]) for _, _, loop in template._loops)


def instantiate_analyzed(template: GraphTemplate, bindings: Mapping[str, int]) -> tuple[ConcreteGraph, LifetimeTable]:
    """``(g, analyze(g))`` for ``g = template.instantiate(bindings)``, served
    from the template's skeleton cache when the trip counts were seen before."""
    b = dict(bindings)
    template.freeze()
    if any(loop.trip_symbol not in b for _, _, loop in template._loops):
        return template.instantiate(b), None  # raises the template's InstantiationError
    key = _trip_key(template, b)
    cache: OrderedDict = template.__dict__.setdefault("_skeletons", OrderedDict())
    sk = cache.get(key)
    if sk is None:
        g = template.instantiate(b)
        table = analyze(g)
        cache[key] = _Skeleton(template, g, table)
        if len(cache) > _MAX_SKELETONS:
            cache.popitem(last=False)
        return g, table
    cache.move_to_end(key)
    # the template validates bindings on instantiate; keep the same contract
    missing = [s for s in template.symbols if s not in b]
    if missing:
        raise InstantiationError(f"missing bindings for symbols {missing}")
    for s in template.symbols:
        if not isinstance(b[s], int) or b[s] < 0:
            raise InstantiationError(f"binding {s}={b[s]!r} is not a non-negative integer")
    return sk.rebind(template, b)
