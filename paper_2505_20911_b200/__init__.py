"""paper_2505_20911_b200 -- B200-native TGV explicit-FD RK time step.

A drop-in for the hot path of the reference solver (mpfd,
/root/reference/proj): per-dataset precision (PrecisionConfig), grid / halo
setup (GridSpec), the residual evaluator and the low-storage RK time-step
driver, executed by hand-written sm_100a CUDA kernels behind the C-ABI in
include/mpfd_b200.h.  This module is the Python mirror of that interface
(names and semantics follow the reference's C++ API); there is no CPU
fallback: importing it without the built extension raises.
"""
from .solver import (  # noqa: F401
    B16, B32, B64, DEFAULT, STORESOME, STRICT, STOREROUND,
    ConfigError, DeviceError, DivergenceEvent, DiagnosticsRecord, AdvanceResult,
    FlowParams, GridSpec, PrecisionConfig, RKScheme, SplitCoefficients, StepConfig,
    Decomposition, Solver, lib, resolve_preset, split_preset, library_path, issue_ceiling,
    LOCAL, NCCL, IPC, gloo_allgather, halo_plan, merge_divergence, merge_diagnostics,
)

__all__ = [
    "B16", "B32", "B64", "DEFAULT", "STORESOME", "STRICT", "STOREROUND",
    "ConfigError", "DeviceError", "DivergenceEvent", "DiagnosticsRecord", "AdvanceResult",
    "FlowParams", "GridSpec", "PrecisionConfig", "RKScheme", "SplitCoefficients",
    "StepConfig", "Decomposition", "Solver", "lib", "resolve_preset", "split_preset",
    "library_path", "issue_ceiling", "LOCAL", "NCCL", "IPC", "gloo_allgather", "halo_plan",
    "merge_divergence", "merge_diagnostics",
]
