"""The per-step planning fast path (skeleton cache + native first-fit) returns
exactly what the reference's instantiate -> analyze -> plan_first_fit chain
returns, for every template family and a spread of bindings."""
from dataclasses import replace

import pytest

from paper_2601_06562_b200 import chunker, liveness, planner, plancache, workload


def _configs():
    toys = workload.toy_configs()
    llada = workload.ModelConfig("llada_8b", 32, 4096, 12288, 32, 126464, 2, 16 << 30, True, "fused", "none")
    out = [("llada_fused", llada), ("llada_mask_only", replace(llada, logits_mode="mask_only")),
           ("dream_shift", replace(llada, name="dream", d_model=3584, vocab_size=152064, shift_mode="in_place",
                                   logits_mode="mask_only"))]
    out += [(n, c) for n, c in toys.items()]
    out += [("toy_shift_concat", replace(toys["toy_shift"], shift_mode="concat"))]
    return out


@pytest.mark.parametrize("name,cfg", _configs(), ids=[n for n, _ in _configs()])
def test_rebind_equals_fresh_instantiation(name, cfg):
    t = workload.build_layer_template(cfg)
    small = "toy" in name
    Ls = [10, 37, 64] if small else [2048, 32768, 131072]
    for K in [(1, 1), (3, 2), (5, 7)]:
        for L in Ls:
            for M in (1, L // 2, L - 1):
                b = {"L": L, "M": M, "K_logits": K[0], "K_FFN": K[1]}
                g1, t1 = plancache.instantiate_analyzed(t, b)
                g0 = t.instantiate(b)
                t0 = liveness.analyze(g0)
                assert g1.ops == g0.ops and g1.sizes == g0.sizes and g1.bindings == g0.bindings
                assert t1 == t0
                assert planner.plan_first_fit(t1) == planner.plan_first_fit(t0)


def test_search_results_unchanged_by_cache():
    cfg = workload.ModelConfig("llada_8b", 32, 4096, 12288, 32, 126464, 2, 16 << 30, True, "mask_only", "none")
    t = workload.build_layer_template(cfg)
    b = {"L": 262144, "M": 131072}
    peak = chunker.evaluate_peak(t, b, chunker.ChunkConfig(1, 1))
    budget = (peak.total_peak + peak.non_chunkable_peak) // 2
    first = chunker.search_bottleneck(t, b, budget)
    again = chunker.search_bottleneck(t, b, budget)  # served from the skeletons
    assert first == again and first.feasible


def test_native_first_fit_matches_python_restatement():
    import random

    def py_first_fit(groups, alignment):
        placed, offs = [], {}
        for g in sorted(groups, key=lambda g: (g.def_index, -g.size, g.id)):
            if g.size == 0:
                offs[g.id] = 0
                continue
            busy = sorted((o, o + p.size) for p, o in placed
                          if p.def_index <= g.last_use_index and g.def_index <= p.last_use_index)
            at = 0
            for lo, hi in busy:
                if at + g.size <= lo:
                    break
                at = max(at, -(-hi // alignment) * alignment)
            offs[g.id] = at
            placed.append((g, at))
        return offs

    rng = random.Random(7)
    for trial in range(200):
        n = rng.randint(0, 60)
        groups = []
        for i in range(n):
            a = rng.randint(0, 40)
            groups.append(liveness.StorageGroup(f"g{i:03d}", rng.choice([0, 1, 100, 256, 1000, rng.randint(1, 5000)]),
                                                "other", a, a + rng.randint(0, 15), ((f"g{i:03d}", None),)))
        table = liveness.LifetimeTable(tuple(groups), 60)
        al = rng.choice([1, 64, 256])
        assert planner.plan_first_fit(table, al).offsets() == py_first_fit(groups, al)
