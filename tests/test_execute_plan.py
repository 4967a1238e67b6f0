"""The reference's canary plan executor (mosaic/vmm.py:188-291) on the sim/os
backends, with the reference's own test cases (tests/test_vmm.py:100-158)
rebuilt on this package's templates, plus the cuda backend (device fills and
checks inside the arena) under the gpu marker."""
from dataclasses import replace

import pytest

from paper_2601_06562_b200 import liveness, planner, vmm, workload
from paper_2601_06562_b200.dims import const
from paper_2601_06562_b200.errors import CapacityError, ExecutionFault
from paper_2601_06562_b200.graph import new_template
from paper_2601_06562_b200.planner import MemoryPlan, PlanEntry


def _graphs():
    toys = workload.toy_configs()
    for name in ("toy_gated", "toy_shift", "toy_moe"):
        t = workload.build_layer_template(toys[name])
        for K in ((1, 1), (2, 3), (5, 2)):
            yield t.instantiate({"L": 10, "M": 8, "K_logits": K[0], "K_FFN": K[1]})
    t = workload.build_layer_template(replace(toys["tiny_llada"], d_model=16, d_ff=128, vocab_size=64))
    for K in ((1, 1), (3, 2)):
        yield t.instantiate({"L": 40, "M": 20, "K_logits": K[0], "K_FFN": K[1]})


def _corrupt():
    t = new_template(())
    t.add_tensor("a", (const(64),), 1)
    t.add_tensor("b", (const(64),), 1)
    t.add_op("make_a", (), ("a",))
    t.add_op("make_b", (), ("b",))
    t.add_op("use", ("a", "b"), ())
    g = t.instantiate({})
    bad = MemoryPlan(alignment=1, workspace_size=64,
                     entries=(PlanEntry("a", 0, 64, 0, 2, "other"), PlanEntry("b", 0, 64, 1, 2, "other")))
    return g, bad


@pytest.mark.parametrize("backend", ["sim", "os"])
def test_execute_plan_clean_on_planned_graphs(backend):
    for g in _graphs():
        plan = planner.plan_first_fit(liveness.analyze(g))
        ws = vmm.reserve(max(plan.workspace_size, 1) + 4096, page_size=4096, backend=backend)
        try:
            ws.commit_to(plan.workspace_size)
            report = vmm.execute_plan(ws, plan, g)
            assert report.ok and report.ops_executed == g.op_count
        finally:
            ws.close()


def test_execute_plan_requires_commitment():
    g = next(_graphs())
    plan = planner.plan_first_fit(liveness.analyze(g))
    ws = vmm.reserve(plan.workspace_size + 4096, page_size=4096)
    with pytest.raises(CapacityError):
        vmm.execute_plan(ws, plan, g)


@pytest.mark.parametrize("backend", ["sim", "os"])
def test_corrupted_plan_detected_with_pair(backend):
    g, bad = _corrupt()
    ws = vmm.reserve(4096, page_size=4096, backend=backend)
    ws.commit_to(64)
    with pytest.raises(ExecutionFault) as info:
        vmm.execute_plan(ws, bad, g)
    assert set(info.value.groups) == {"a", "b"}
    report = vmm.execute_plan(ws, bad, g, raise_on_fault=False)
    assert not report.ok and report.faults[0].kind == "clobber" and report.faults[0].partner == "b"
    ws.close()


def test_execution_report_json_shape():
    g = next(_graphs())
    plan = planner.plan_first_fit(liveness.analyze(g))
    ws = vmm.reserve(plan.workspace_size + 4096, page_size=4096)
    ws.commit_to(plan.workspace_size)
    d = vmm.execute_plan(ws, plan, g).to_json_dict()
    assert set(d) == {"ops_executed", "faults", "committed_bytes", "workspace_size"}


@pytest.mark.gpu
def test_execute_plan_cuda_arena(native_lib):
    """Device canaries in the cuMem arena: every planned step graph runs clean;
    the overlapping plan faults on the same pair."""
    t = workload.build_layer_template(workload.toy_configs()["tiny_llada"])
    ws = vmm.reserve(1 << 30, backend="cuda")
    try:
        for K in ((1, 1), (3, 2), (7, 5)):
            g = t.instantiate({"L": 2048, "M": 1024, "K_logits": K[0], "K_FFN": K[1]})
            plan = planner.plan_first_fit(liveness.analyze(g))
            ws.commit_to(plan.workspace_size)
            report = vmm.execute_plan(ws, plan, g)
            assert report.ok and report.ops_executed == g.op_count
        g, bad = _corrupt()
        with pytest.raises(ExecutionFault) as info:
            vmm.execute_plan(ws, bad, g)
        assert set(info.value.groups) == {"a", "b"}
    finally:
        ws.close()
