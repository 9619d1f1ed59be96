"""B200-native MLFMA evaluation (drop-in for the evaluation phase of the
reference hfmm engine, arXiv 2006.15367).  See DESIGN.md."""
from .hfmm import (LEDGER_PHASES, AlignPolicy, EvalResult, GlobalSetup, Phase, RankEngine, RunConfig,
                   SchedulerKind, World, build_setup, direct_potential, evaluate_potential,
                   evaluate_with_setup, generate_inputs, resample_matrix)
from ._native import (CudaError, DomainError, HfmmError, InvalidArgument, LengthError, LogicError,
                      NoDeviceError, OutOfRange)

__all__ = [
    "LEDGER_PHASES", "AlignPolicy", "EvalResult", "GlobalSetup", "Phase", "RankEngine", "RunConfig",
    "SchedulerKind", "World",
    "build_setup", "direct_potential", "evaluate_potential", "evaluate_with_setup", "generate_inputs",
    "resample_matrix",
    "CudaError", "DomainError", "HfmmError", "InvalidArgument", "LengthError", "LogicError",
    "NoDeviceError", "OutOfRange",
]
