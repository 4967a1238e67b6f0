"""B200-native mask-only logits + remask hot path of Mosaic (arXiv 2601.06562).

Name-compatible with the reference package ``mosaic`` (mosaic/__init__.py:9-43):
``GatherGemmProblem`` / ``gather_gemm`` run on sm_100a kernels through the C
ABI in ``include/mosaic_b200.h``; the fused production entry points are
:func:`gather_logits_stats` and :class:`MaskOnlyHead`; the graph registrar,
liveness, first-fit planner, chunk search and step loop keep the reference
interfaces and drive the device executor.
"""
from .errors import (
    AnalysisError,
    BuildError,
    CapacityError,
    DeviceError,
    ExecutionFault,
    InfeasibleRunError,
    InputError,
    InstantiationError,
    MosaicError,
    ParseError,
    ResourceError,
    TooLarge,
    UsageError,
    ValidationError,
)
from .chunker import ChunkConfig, PeakReport, SearchOutcome, evaluate_peak, search_bottleneck, search_bruteforce
from .dims import Dim, ceildiv, const, parse_dim, sym
from .graph import ConcreteGraph, GraphTemplate, load_template, new_template, template_from_json_dict
from .liveness import LifetimeTable, StorageGroup, analyze, max_live
from .planner import MemoryPlan, PlanStats, plan_exact, plan_first_fit, validate
from .vmm import ExecutionReport, Fault, Workspace, commit_to, execute_plan, reserve
from .workload import (
    ModelConfig,
    MoEConfig,
    ScenarioConfig,
    build_layer_template,
    find_lmax,
    load_model_config,
    par_curve,
    simulate_run,
    toy_configs,
)
from .kernel import (
    GatherGemmProblem,
    ScratchAccount,
    dense_then_discard,
    gather_gemm,
    gather_logits_stats,
    gemm_reference,
)
from .hotpath import MaskOnlyHead, StepOutput

__version__ = "0.1.0"
