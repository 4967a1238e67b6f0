"""CPU checks of the MoE expert-FFN extension: the routing restatement in the
oracle (closed form; UNPINNED by the reference, which has no routing) and the
executable MoE template registered through the reference's graph API."""
from dataclasses import replace

import numpy as np
import pytest

import mosaic_oracle as orc


def test_route_closed_form_small():
    z = np.array([[0.0, 2.0, 1.0, 2.0],   # tie 1 vs 3 -> 1 first
                  [5.0, -1.0, 5.0, 5.0]])  # three-way tie -> 0, 2
    r = orc.moe_route(z, 2)
    assert r["experts"].tolist() == [[1, 3], [0, 2]]
    # dispatch order (expert, row, j): e0 <- (1,0); e1 <- (0,0); e2 <- (1,1); e3 <- (0,1)
    assert r["disp_row"].tolist() == [1, 0, 1, 0]
    assert r["comb_pos"].tolist() == [[1, 3], [0, 2]]
    assert r["expert_off"].tolist() == [0, 1, 2, 3, 4]
    assert np.allclose(r["comb_w"], 0.5)


@pytest.mark.parametrize("rows,E,k", [(50, 8, 2), (200, 64, 8), (17, 5, 5)])
def test_route_properties(rows, E, k):
    rng = np.random.default_rng(rows)
    z = rng.standard_normal((rows, E))
    r = orc.moe_route(z, k, row_base=100)
    assert np.allclose(r["comb_w"].sum(axis=1), 1.0)
    assert np.all(np.diff(r["comb_w"], axis=1) <= 1e-15)  # weights follow logit order
    off = r["expert_off"]
    assert off[0] == 0 and off[-1] == rows * k and np.all(np.diff(off) >= 0)
    # every (row, j) lands in its expert's segment, rows ascending inside a segment
    for e in range(E):
        seg = r["disp_row"][off[e]:off[e + 1]]
        assert np.all(np.diff(seg) > 0)
    pos = r["comb_pos"]
    assert sorted(pos.reshape(-1).tolist()) == list(range(rows * k))
    assert np.array_equal(r["disp_row"][pos] - 100, np.repeat(np.arange(rows)[:, None], k, axis=1))
    for rr in range(rows):
        for j in range(k):
            e = r["experts"][rr, j]
            assert off[e] <= pos[rr, j] < off[e + 1]


def test_combine_closed_form():
    src = np.arange(12, dtype=np.float64).reshape(6, 2)
    pos = np.array([[5, 0], [2, 3], [1, 4]])
    w = np.array([[0.5, 0.5], [1.0, 0.0], [0.25, 0.75]])
    out = orc.moe_combine(src, pos, w)
    assert out.tolist() == [[5.0, 6.0], [4.0, 5.0], [6.5, 7.5]]


def test_moe_template_registers_routing_in_the_ffn_loop():
    from paper_2601_06562_b200 import chunker, workload

    cfg = workload.toy_configs()["tiny_moe"]
    t = workload.build_layer_template(cfg)
    g = t.instantiate({"L": 2048, "M": 1024, "K_logits": 1, "K_FFN": 4})
    kinds = [op.kind for op in g.ops if op.op_id.startswith("l0.")]
    assert kinds.count("moe_route") == 4 and kinds.count("moe_combine") == 4
    # chunk tensors scale with ceil(L/K) * top_k rows
    assert t.instance_shape("l0.xin", g.bindings) == (512 * 2, 256)
    assert t.instance_shape("l0.act", g.bindings) == (512 * 2, 128)
    assert "l0.up" not in t.tensors and "l0.gate" not in t.tensors  # K10's SwiGLU epilogue writes act only
    assert t.instance_shape("l0.expert_off", g.bindings) == (9,)
    # the search chunks the MoE FFN when it is the bottleneck (wider experts, top-4)
    t = workload.build_layer_template(replace(cfg, d_ff=512, moe=workload.MoEConfig(8, 4)))
    peak1 = chunker.evaluate_peak(t, {"L": 8192, "M": 4096}, chunker.ChunkConfig(1, 1))
    assert peak1.bottleneck == "ffn"
    budget = (peak1.total_peak + peak1.non_chunkable_peak) // 2  # above the attention floor
    out = chunker.search_bottleneck(t, {"L": 8192, "M": 4096}, budget)
    assert out.config.k_ffn > 1 and out.reason == "fits"


def test_moe_template_first_fit_is_tight_and_in_place():
    from paper_2601_06562_b200 import liveness, planner, workload

    cfg = workload.toy_configs()["tiny_moe"]
    g = workload.build_layer_template(cfg).instantiate({"L": 4096, "M": 2048, "K_logits": 2, "K_FFN": 3})
    table = liveness.analyze(g)
    plan = planner.plan_first_fit(table)
    planner.validate(plan, table)
    assert plan.workspace_size == liveness.max_live(table)
    grp = {m: gr.id for gr in table.groups for m in gr.members}
    assert grp[("l0.down_e", 0)] == grp[("l0.xin", 0)]   # down writes over the dispatch rows
    assert ("l0.act", 1) in grp


def test_reference_modes_keep_the_reference_moe_template():
    """mask_only/eager MoE templates stay the reference's (plans pinned to it);
    the executor refuses them rather than guessing a routing."""
    import torch

    from paper_2601_06562_b200 import workload
    from paper_2601_06562_b200.errors import InputError
    from paper_2601_06562_b200.executor import RandomDLLM

    cfg = replace(workload.toy_configs()["tiny_moe"], logits_mode="mask_only")
    ops = {op.kind for op in workload.build_layer_template(cfg).ops}
    assert "moe_route" not in ops and "ffn_up" in ops
    with pytest.raises(InputError):
        RandomDLLM(cfg, torch.device("cpu"))


def test_fused_gather_template_drops_the_compacted_buffer():
    from paper_2601_06562_b200 import chunker, workload

    base = workload.toy_configs()["tiny_llada"]
    t_f = workload.build_layer_template(base)
    t_g = workload.build_layer_template(replace(base, logits_mode="fused_gather"))
    assert "hc" in t_f.tensors and "hc" not in t_g.tensors
    kinds = {op.kind for op in t_g.ops}
    assert "lmhead_stats_gather" in kinds and "gather" not in kinds
    b = {"L": 4096, "M": 4000}
    pf = chunker.evaluate_peak(t_f, b, chunker.ChunkConfig(1, 1))
    pg = chunker.evaluate_peak(t_g, b, chunker.ChunkConfig(1, 1))
    assert pg.component_peaks["logits"] < pf.component_peaks["logits"]
    assert pg.total_peak <= pf.total_peak


def test_fused_ffn_template_holds_act_only():
    from paper_2601_06562_b200 import chunker, workload

    base = workload.toy_configs()["tiny_llada"]
    t0 = workload.build_layer_template(base)
    t1 = workload.build_layer_template(replace(base, fused_ffn=True))
    assert {"l0.up", "l0.gate"} <= set(t0.tensors) and not ({"l0.up", "l0.gate"} & set(t1.tensors))
    assert any(op.kind == "ffn_gate_up" for op in t1.ops)
    b = {"L": 8192, "M": 4096}
    p0 = chunker.evaluate_peak(t0, b, chunker.ChunkConfig(1, 1))
    p1 = chunker.evaluate_peak(t1, b, chunker.ChunkConfig(1, 1))
    assert p1.component_peaks["ffn"] * 2 == p0.component_peaks["ffn"]  # [L, d_ff] once instead of twice
    # the residual epilogue: no `down` chunk rows, no [L, d] ffn_acc
    assert not ({"l0.down", "l0.ffn_acc"} & set(t1.tensors)) and any(op.kind == "ffn_down_res" for op in t1.ops)
    assert p1.total_peak < p0.total_peak
    assert workload.model_config_from_json_dict(replace(base, fused_ffn=True).to_json_dict()).fused_ffn
