"""Property tests (hypothesis) of the CPU restatements and the host control
plane: the algebra the GPU path relies on, checked over generated inputs
rather than fixed cases. Oracle functions cite the reference lines they
restate (oracle/mosaic_oracle.py); the planner and liveness are this package's
reimplementations of mosaic/planner.py:107-142 and mosaic/liveness.py:43-154.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "oracle"))
import mosaic_oracle as orc  # noqa: E402

SETTINGS = settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])


def _logits(seed: int, rows: int, cols: int, ties: bool) -> np.ndarray:
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((rows, cols)) * 3.0
    if ties:  # coarse grid: many exact ties inside and across splits
        z = np.round(z)
    return z


@SETTINGS
@given(seed=st.integers(0, 2**31 - 1), rows=st.integers(1, 9), cols=st.integers(1, 70),
       n_cuts=st.integers(0, 6), ties=st.booleans())
def test_split_merge_equals_whole_row(seed, rows, cols, n_cuts, ties):
    """K3 splits + K4 merge (any contiguous split of the vocabulary, fixed
    order) give the whole row's max, sum-exp and argmax with the lowest-index
    tie rule."""
    z = _logits(seed, rows, cols, ties)
    rng = np.random.default_rng(seed + 1)
    cuts = sorted(set(rng.integers(1, cols, size=n_cuts).tolist())) if cols > 1 else []
    bounds = [0] + cuts + [cols]
    m, s, a = orc.merge_triples(orc.split_stats(z, bounds))
    whole = orc.softmax_stats(z)
    assert np.array_equal(m, whole["max"])
    assert np.array_equal(a, whole["arg"])
    assert np.allclose(s, whole["sum"], rtol=1e-12)


@SETTINGS
@given(seed=st.integers(0, 2**31 - 1), rows=st.integers(1, 6), cols=st.integers(2, 40),
       n_parts=st.integers(2, 5), ties=st.booleans())
def test_merge_is_order_independent_on_max_and_arg(seed, rows, cols, n_parts, ties):
    """The rank / split merge is associative and commutative on (max, argmax)
    and on the sum up to rounding, so the vocab-sharded exchange can merge in
    any fixed order."""
    z = _logits(seed, rows, cols, ties)
    bounds = np.linspace(0, cols, n_parts + 1).astype(int).tolist()
    bounds = sorted(set(bounds))
    parts = orc.split_stats(z, bounds)
    m1, s1, a1 = orc.merge_triples(parts)
    m2, s2, a2 = orc.merge_triples(parts[::-1])
    assert np.array_equal(m1, m2) and np.array_equal(a1, a2)
    assert np.allclose(s1, s2, rtol=1e-12)


@SETTINGS
@given(seed=st.integers(0, 2**31 - 1), M=st.integers(0, 60), k=st.integers(-2, 70),
       levels=st.integers(1, 8))
def test_remask_select_rule(seed, M, k, levels):
    """K5's rule: exactly min(max(k, 0), M) rows; every kept row is at least as
    confident as every dropped row; among equal float32 confidences the lower
    position wins."""
    rng = np.random.default_rng(seed)
    conf = rng.integers(1, levels + 1, size=M).astype(np.float32) / levels  # many exact ties
    pos = np.sort(rng.choice(10 * M + 1, size=M, replace=False)) if M else np.zeros(0, np.int64)
    sel = orc.remask_select(conf, pos, k)
    assert int(sel.sum()) == max(0, min(k, M))
    if sel.any() and (~sel).any():
        assert conf[sel].min() >= conf[~sel].max()
        edge = conf[sel].min()
        if (conf[~sel] == edge).any():
            assert pos[sel & (conf == edge)].max() < pos[~sel & (conf == edge)].min()


@SETTINGS
@given(seed=st.integers(0, 2**31 - 1), L=st.integers(0, 300), p=st.floats(0.0, 1.0))
def test_mask_compact_is_ascending_flatnonzero(seed, L, p):
    """K1's restatement: ascending positions of the mask id, nothing else."""
    rng = np.random.default_rng(seed)
    x = rng.integers(0, 50, size=L).astype(np.int32)
    x[rng.random(L) < p] = 49
    idx = orc.mask_compact(x, 49)
    assert np.array_equal(idx, np.flatnonzero(x == 49))
    assert np.all(np.diff(idx) > 0)


@SETTINGS
@given(L=st.integers(1, 5000), rp=st.sampled_from([0.0, 0.25, 0.5, 0.7]), steps=st.integers(1, 80))
def test_unmask_counts_commit_everything(L, rp, steps):
    """The per-step counts from the banker's-rounding schedule are
    non-negative and sum to the output length (mosaic/workload.py:140-146)."""
    ks = orc.unmask_counts(L, rp, steps)
    assert all(k >= 0 for k in ks)
    assert sum(ks) == orc.output_length(L, rp)


@SETTINGS
@given(seed=st.integers(0, 2**31 - 1), rows=st.integers(1, 40), E=st.integers(2, 16), data=st.data())
def test_moe_route_dispatch_tables(seed, rows, E, data):
    """K8's restatement: top-k per row by (logit desc, expert asc), weights a
    softmax over the chosen logits, dispatch slots grouped by expert in
    ascending (row, j) order, and comb_pos inverting disp_row."""
    k = data.draw(st.integers(1, E))
    rng = np.random.default_rng(seed)
    z = np.round(rng.standard_normal((rows, E)) * 2, 1)  # ties between experts
    r = orc.moe_route(z, k)
    sel, off = r["experts"], r["expert_off"]
    assert np.all(np.diff(off) >= 0) and off[-1] == rows * k
    for i in range(rows):
        chosen = set(sel[i].tolist())
        assert len(chosen) == k
        worst = min(z[i, e] for e in chosen)
        for e in range(E):  # nothing better (or equal with a lower id) was left out
            if e not in chosen:
                assert z[i, e] < worst or (z[i, e] == worst and e > max(c for c in chosen if z[i, c] == worst))
    assert np.allclose(r["comb_w"].sum(axis=1), 1.0)
    flat_e = sel.reshape(-1)
    for slot in range(rows * k):  # slot -> (row, j) and back
        row = r["disp_row"][slot]
        j = int(np.flatnonzero(r["comb_pos"][row] == slot)[0])
        e = flat_e[row * k + j]
        assert off[e] <= slot < off[e + 1]
    for e in range(E):  # inside an expert segment: ascending (row, j)
        seg = [int(r["disp_row"][s]) for s in range(off[e], off[e + 1])]
        assert seg == sorted(seg)


def _random_table(seed: int, n: int, length: int):
    from paper_2601_06562_b200.liveness import LifetimeTable, StorageGroup

    rng = np.random.default_rng(seed)
    groups = []
    for i in range(n):
        a = int(rng.integers(0, length))
        b = int(rng.integers(a, length))
        groups.append(StorageGroup(id=f"g{i}", size=int(rng.integers(1, 5000)), tag="other", def_index=a,
                                   last_use_index=b, members=((f"g{i}", None),)))
    return LifetimeTable(groups=tuple(groups), length=length)


@SETTINGS
@given(seed=st.integers(0, 2**31 - 1), n=st.integers(1, 40), length=st.integers(1, 30),
       align=st.sampled_from([1, 64, 256]))
def test_native_first_fit_is_valid_and_aligned(seed, n, length, align):
    """The native first-fit (C++, csrc/planner.cu; mosaic/planner.py:107-142
    semantics) never overlaps two groups that are live together, aligns every
    offset, and its workspace is the highest end offset."""
    from paper_2601_06562_b200 import planner

    table = _random_table(seed, n, length)
    plan = planner.plan_first_fit(table, alignment=align)
    offs = plan.offsets()
    gs = {g.id: g for g in table.groups}
    assert all(o % align == 0 for o in offs.values())
    ends = [offs[g] + gs[g].size for g in offs]
    assert plan.workspace_size >= max(ends)
    ids = list(offs)
    for i, a in enumerate(ids):
        for b in ids[i + 1:]:
            ga, gb = gs[a], gs[b]
            live = not (ga.last_use_index < gb.def_index or gb.last_use_index < ga.def_index)
            if live:
                assert offs[a] + ga.size <= offs[b] or offs[b] + gb.size <= offs[a]
    assert planner.validate(plan, table).ok
