"""The CPU oracle pinned against the reference's own outputs (tests/golden) and
the reference's known-answer tests (tests/test_kernel.py of the reference)."""
import json

import numpy as np
import pytest

import mosaic_oracle as orc
from conftest import GOLDEN


@pytest.fixture(scope="module")
def kg():
    return np.load(GOLDEN / "kernel_golden.npz")


def test_gather_gemm_matches_reference_bitwise(kg):
    cases = sorted({k.split("_")[0] for k in kg.files if k.startswith("rand")})
    assert len(cases) == 40
    for c in cases:
        h, w, idx, tiles = kg[c + "_hidden"], kg[c + "_weight"], kg[c + "_idx"], kg[c + "_tiles"]
        out = orc.gather_gemm(h, w, idx.tolist(), *map(int, tiles))
        assert np.array_equal(out, kg[c + "_out"]), c


def test_bf16_case_matches_reference(kg):
    out = orc.gather_gemm(kg["bf16case_hidden"], kg["bf16case_weight"], kg["bf16case_idx"].tolist())
    assert np.array_equal(out, kg["bf16case_out"])
    # the BLAS form used at large shapes agrees to fp64 rounding
    blas = orc.logits_f64(orc.gather_rows(kg["bf16case_hidden"], kg["bf16case_idx"]),
                          kg["bf16case_weight"].T)
    assert np.allclose(blas, kg["bf16case_out"], rtol=1e-12, atol=1e-12)


def test_known_answers():
    # reference tests/test_kernel.py:15-35
    hidden = np.arange(12, dtype=np.float64).reshape(4, 3)
    assert np.array_equal(orc.gather_gemm(hidden, np.eye(3), (2, 0)), hidden[[2, 0], :])
    out = orc.gather_gemm(np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]]), np.eye(2), (1,))
    assert np.array_equal(out, np.array([[3.0, 4.0]]))
    assert np.array_equal(orc.gemm_reference([[2.0]], [[3.0]]), np.array([[6.0]]))
    rng = np.random.default_rng(52)
    h = rng.standard_normal((13, 9))
    w = rng.standard_normal((9, 21))
    assert np.allclose(orc.gather_gemm(h, w, tuple(range(13))), orc.dense_then_discard(h, w, range(13)),
                       rtol=1e-12, atol=0)


def test_tile_invariance_bitwise():
    rng = np.random.default_rng(51)
    h = rng.standard_normal((23, 17))
    w = rng.standard_normal((17, 29))
    idx = tuple(int(i) for i in rng.choice(23, size=11, replace=False))
    outs = [orc.gather_gemm(h, w, idx, *t) for t in ((1, 1, 1), (2, 5, 3), (7, 7, 7), (64, 64, 64))]
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)


def test_schedule_matches_reference():
    cases = json.loads((GOLDEN / "sched_golden.json").read_text())
    for c in cases:
        L, rp, N = c["L"], c["prompt_ratio"], c["steps"]
        assert orc.output_length(L, rp) == c["output_length"]
        assert [orc.masked_at(L, rp, N, n) for n in range(N + 1)] == c["masked_at"]
        k = orc.unmask_counts(L, rp, N)
        assert sum(k) == c["output_length"] and all(v >= 0 for v in k)
    # SURVEY §8a a10 worked examples (banker's rounding: 7.5 -> 8, 2.5 -> 2)
    assert orc.unmask_counts(10, 0.0, 4) == [2, 3, 3, 2]
    assert orc.unmask_counts(65536, 0.5, 48)[:4] == [683, 682, 683, 683]


def test_mask_compact_and_validate():
    x = np.array([5, 9, 9, 1, 9, 0], dtype=np.int32)
    assert orc.mask_compact(x, 9).tolist() == [1, 2, 4]
    assert orc.mask_compact(x, 7).tolist() == []
    with pytest.raises(ValueError):
        orc.validate_mask_idx(4, [0, 0])
    with pytest.raises(ValueError):
        orc.validate_mask_idx(4, [4])


def test_stats_split_merge_equals_whole_row():
    rng = np.random.default_rng(3)
    z = rng.standard_normal((50, 1000)) * 3
    whole = orc.softmax_stats(z)
    bounds = [0, 256, 300, 777, 1000]
    m, s, a = orc.merge_triples(orc.split_stats(z, bounds))
    assert np.allclose(m, whole["max"]) and np.allclose(s, whole["sum"], rtol=1e-12)
    assert np.array_equal(a, whole["arg"])
    assert np.allclose(whole["conf"], np.exp(z[np.arange(50), whole["arg"]] - whole["lse"]))


def test_argmax_ties_take_lowest_index():
    z = np.zeros((1, 10))
    z[0, [3, 7]] = 5.0
    assert orc.softmax_stats(z)["arg"][0] == 3
    parts = orc.split_stats(z, [0, 5, 10])
    parts_rev = [parts[1], parts[0]]
    assert orc.merge_triples(parts)[2][0] == 3
    assert orc.merge_triples(parts_rev)[2][0] == 3


def test_remask_select_rule():
    conf = np.array([0.5, 0.9, 0.5, 0.1, 0.9], dtype=np.float32)
    pos = np.array([10, 40, 5, 7, 30])
    sel = orc.remask_select(conf, pos, 3)
    # 0.9@30, 0.9@40, then 0.5 tie broken by lower position (5)
    assert sel.tolist() == [False, True, True, False, True]
    assert orc.remask_select(conf, pos, 0).sum() == 0
    assert orc.remask_select(conf, pos, 99).sum() == 5
    x = np.array([0] * 50)
    out = orc.commit(x, pos, np.array([1, 2, 3, 4, 5]), sel)
    assert out[40] == 2 and out[5] == 3 and out[30] == 5 and out[10] == 0


def test_bf16_round():
    a = np.array([1.0, 1.00390625, 1.005859375, -3.14159, 65504.0])
    r = orc.bf16_round(a)
    assert r[0] == 1.0 and r[1] == 1.0  # tie to even
    assert r[2] == 1.0078125
    assert abs(r[3] - -3.140625) < 1e-9
    bits = orc.bf16_bits(np.array([1.0, -2.0]))
    assert bits.tolist() == [0x3F80, 0xC000]


def test_full_step_small():
    rng = np.random.default_rng(4)
    L, d, V, mask_id = 64, 16, 40, 39
    x = rng.integers(0, 30, size=L).astype(np.int32)
    x[rng.choice(L, 20, replace=False)] = mask_id
    H = rng.standard_normal((L, d))
    W = rng.standard_normal((V, d)) * 0.3
    out = orc.step(x, H, W, mask_id, k=5)
    assert out["selected"].sum() == 5
    assert (out["x"] == mask_id).sum() == 15
    # the committed tokens are the argmax of the oracle logits at those positions
    z = orc.logits_f64(H[out["idx"]], W)
    assert np.array_equal(out["arg"], z.argmax(1))
