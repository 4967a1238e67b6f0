"""The control plane (registrar, liveness, planner, chunk search, step loop,
L_max) pinned against fixtures produced by the reference package itself
(oracle/make_golden_control.py). Exact equality everywhere: these are integer
algorithms."""
import json
from dataclasses import replace

import pytest

from conftest import GOLDEN
from paper_2601_06562_b200 import chunker, dims, graph, liveness, planner, workload
from paper_2601_06562_b200.errors import (AnalysisError, BuildError, InfeasibleRunError,
                                          InstantiationError, MosaicError, ParseError)

G = json.loads((GOLDEN / "control_golden.json").read_text())
SMALL = [n for n in G["models"] if n.startswith("toy") or n == "tiny_llada"]
BIG = [n for n in G["models"] if n not in SMALL]


def cfg_of(name):
    return workload.model_config_from_json_dict(G["models"][name]["config"])


def k(x):
    return (x[0], x[1])


# --------------------------------------------------------------------------- dims
def test_dims_render_and_eval():
    env = {"L": 37, "M": 5, "K": 4, "K_FFN": 3, "d": 7, "a": 2, "b": 3, "c": 4}
    for case in G["dims"]:
        d = dims.parse_dim(case["text"])
        assert str(d) == case["str"]
        assert d.eval(env) == case["eval"]
        assert str(dims.parse_dim(str(d))) == case["str"]


def test_dims_errors():
    for bad in ("", "L+", "ceil(L)", "L $ M", "(L", "ceil", "L M"):
        with pytest.raises(ParseError):
            dims.parse_dim(bad)
    with pytest.raises(InstantiationError):
        dims.sym("Q").eval({})
    with pytest.raises(InstantiationError):
        dims.ceildiv("L", "K").eval({"L": 3, "K": 0})
    assert dims.ceil_div(7, 2) == 4 and dims.ceil_div(0, 5) == 0
    with pytest.raises(ParseError):
        dims.const(-1)


# --------------------------------------------------------------------------- templates
@pytest.mark.parametrize("name", list(G["models"]))
def test_template_structure_matches_reference(name):
    cfg = cfg_of(name)
    for variant, v in G["models"][name]["variants"].items():
        lm, sm = variant.split("/")
        t = workload.build_layer_template(replace(cfg, logits_mode=lm, shift_mode=sm))
        assert t.to_json_dict() == v["template"], variant
        # and the reference JSON loads through our registrar unchanged
        t2 = graph.template_from_json_dict(v["template"])
        assert t2.to_json_dict() == v["template"]


def _graph_dump(g):
    ks = lambda x: [x[0], x[1]]  # noqa: E731
    return {
        "ops": [[o.op_id, o.iteration, o.kind, [ks(a) for a in o.inputs], [ks(a) for a in o.outputs],
                 [[ks(a), ks(b)] for a, b in o.in_place]] for o in g.ops],
        "sizes": sorted([[a[0], a[1], v] for a, v in g.sizes.items()],
                        key=lambda x: (x[0], -1 if x[1] is None else x[1])),
        "aliases": [[ks(a), ks(b)] for a, b in g.aliases],
        "barriers": [[[ks(a) for a in m], r] for m, r in g.barriers],
        "loop_symbol": sorted([[a[0], a[1], v] for a, v in g.loop_symbol.items()]),
    }


@pytest.mark.parametrize("name", SMALL)
def test_instantiate_analyze_plan_small(name):
    cfg = cfg_of(name)
    for variant, v in G["models"][name]["variants"].items():
        lm, sm = variant.split("/")
        t = workload.build_layer_template(replace(cfg, logits_mode=lm, shift_mode=sm))
        for inst in v["instances"]:
            L, M, kl, kf = inst["bind"]
            g = t.instantiate({"L": L, "M": M, "K_logits": kl, "K_FFN": kf})
            assert _graph_dump(g) == inst["graph"], (variant, inst["bind"])
            tab = liveness.analyze(g)
            got = [[x.id, x.size, x.tag, x.def_index, x.last_use_index, [list(m) for m in x.members],
                    x.chunkable_symbol] for x in tab.groups]
            assert got == inst["table"]["groups"] and tab.length == inst["table"]["length"]
            assert liveness.live_profile(tab) == inst["profile"]
            assert liveness.dominant_tags(tab) == inst["dominant"]
            p = planner.plan_first_fit(tab)
            assert p.offsets() == inst["offsets"] and p.workspace_size == inst["workspace"]
            assert liveness.max_live(tab) == inst["max_live"]
            assert planner.validate(p, tab).ok


@pytest.mark.parametrize("name", BIG)
def test_plan_and_peak_report_big(name):
    cfg = cfg_of(name)
    for variant, v in G["models"][name]["variants"].items():
        lm, sm = variant.split("/")
        t = workload.build_layer_template(replace(cfg, logits_mode=lm, shift_mode=sm))
        for inst in v["instances"]:
            L, M, kl, kf = inst["bind"]
            g = t.instantiate({"L": L, "M": M, "K_logits": kl, "K_FFN": kf})
            assert len(g.ops) == inst["op_count"]
            tab = liveness.analyze(g)
            p = planner.plan_first_fit(tab)
            assert p.offsets() == inst["offsets"]
            assert p.workspace_size == inst["workspace"] and liveness.max_live(tab) == inst["max_live"]
            r = chunker.evaluate_peak(t, {"L": L, "M": M}, chunker.ChunkConfig(kl, kf))
            assert r.__dict__ == inst["report"]


@pytest.mark.parametrize("name", list(G["models"]))
def test_chunk_search_matches_reference(name):
    cfg = cfg_of(name)
    for variant, v in G["models"][name]["variants"].items():
        lm, sm = variant.split("/")
        t = workload.build_layer_template(replace(cfg, logits_mode=lm, shift_mode=sm))
        L, M = v["instances"][0]["bind"][:2]
        for s in v["searches"]:
            out = chunker.search_bottleneck(t, {"L": L, "M": M}, s["budget"], k_cap=48)
            assert out.to_json_dict() == s["bottleneck"], (variant, s["budget"])
            if "brute" in s:
                b = chunker.search_bruteforce(t, {"L": L, "M": M}, s["budget"], k_max=8)
                assert b.to_json_dict() == s["brute"]


@pytest.mark.parametrize("name", SMALL)
def test_simulate_run_matches_reference(name):
    cfg = cfg_of(name)
    exp = G["models"][name]["simulate"]
    scen = workload.ScenarioConfig(10 if name.startswith("toy") else 2048, 0.5, 4,
                                   budget=cfg.weights_bytes + 4000 if name.startswith("toy") else None)
    if isinstance(exp, dict):
        with pytest.raises(InfeasibleRunError) as e:
            workload.simulate_run(cfg, scen)
        assert e.value.step_index == exp["infeasible"]
        return
    res = workload.simulate_run(cfg, scen)
    got = [{"masked": r.state.masked_count, "par": r.metrics.par, "peak_component": r.metrics.peak_component,
            "theoretical_peak": r.metrics.theoretical_peak, "k": [r.metrics.k_logits, r.metrics.k_ffn],
            "trace_peak": r.trace.peak, "trace_avg": r.trace.average} for r in res]
    assert got == exp


@pytest.mark.parametrize("name", [n for n in SMALL if n.startswith("toy")])
def test_find_lmax_matches_reference(name):
    cfg = cfg_of(name)
    lm = G["models"][name]["lmax"]
    for key_, feats in (("global", ("global_plan",)), ("global_mask", ("global_plan", "mask_only")),
                        ("global_mask_chunk", ("global_plan", "mask_only", "chunking"))):
        want = lm[key_]
        if isinstance(want, dict):
            with pytest.raises(MosaicError):
                workload.find_lmax(cfg, 0.5, lm["budget"], feats, l_cap=4096)
        else:
            assert workload.find_lmax(cfg, 0.5, lm["budget"], feats, l_cap=4096) == want


def test_random_graphs_liveness_and_first_fit():
    assert len(G["random_graphs"]) >= 20
    for case in G["random_graphs"]:
        t = graph.template_from_json_dict(case["template"])
        g = t.instantiate(case["bindings"])
        tab = liveness.analyze(g)
        got = [[x.id, x.size, x.tag, x.def_index, x.last_use_index, [list(m) for m in x.members],
                x.chunkable_symbol] for x in tab.groups]
        assert got == case["table"]["groups"], case["seed"]
        p = planner.plan_first_fit(tab, alignment=64)
        assert p.offsets() == case["offsets"] and p.workspace_size == case["workspace"]
        if case["exact_ws"] is not None:
            ex = planner.plan_exact(tab, alignment=64)
            assert ex.workspace_size == case["exact_ws"], case["seed"]
            assert planner.validate(ex, tab).ok


# --------------------------------------------------------------------------- builder errors
def test_registrar_rejects_malformed_templates():
    t = graph.new_template(("L", "K"))
    t.add_tensor("x", ("L",), 4, graph_input=True)
    t.add_tensor("y", ("L",), 4)
    with pytest.raises(BuildError):
        t.add_tensor("y", ("L",), 4)
    with pytest.raises(BuildError):
        t.add_tensor("z", ("Q",), 4)
    with pytest.raises(BuildError):
        t.add_tensor("z", ("L",), 0)
    with pytest.raises(BuildError):
        t.add_tensor("z", ("L",), 4, tag="nope")
    with pytest.raises(BuildError):
        t.add_op("o", ("y",), ())  # y not produced yet
    t.add_op("o1", ("x",), ("y",))
    with pytest.raises(BuildError):
        t.add_op("o2", ("x",), ("y",))  # produced twice
    with pytest.raises(BuildError):
        t.add_op("o1", (), ())
    with pytest.raises(BuildError):
        t.add_op("o3", ("x",), ("x",))  # graph input as output
    t.add_tensor("w", ("L",), 4)
    with pytest.raises(BuildError):
        t.add_op("o4", ("x",), ("w",), in_place={"w": "x"})  # reuse of graph input
    with pytest.raises(BuildError):
        t.add_chunk_loop(("o1",), "Z")
    with pytest.raises(BuildError):
        t.add_alias("y", "y")
    t.freeze()
    with pytest.raises(BuildError):
        t.add_tensor("q", ("L",), 4)
    with pytest.raises(InstantiationError):
        t.instantiate({"L": 3})
    with pytest.raises(InstantiationError):
        t.instantiate({"L": -1, "K": 1})


def test_liveness_errors():
    t = graph.new_template(())
    t.add_tensor("a", (4,), 1)
    t.add_tensor("b", (4,), 1)
    t.add_op("p", (), ("a",))
    t.add_op("q", ("a",), ("b",), in_place={"b": "a"})
    t.add_alias("b", "a")  # closes a cycle with the in_place edge
    with pytest.raises(AnalysisError):
        liveness.analyze(t.instantiate({}))
