"""B200-native mask-only logits + remask hot path of Mosaic (arXiv 2601.06562).

Name-compatible with the reference package ``mosaic`` (mosaic/__init__.py:9-43)
for the hot path: ``GatherGemmProblem`` / ``gather_gemm`` run on sm_100a
kernels through the C ABI in ``include/mosaic_b200.h``; the fused production
entry points are :func:`gather_logits_stats` and :class:`MaskOnlyHead`.
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
