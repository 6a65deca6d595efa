"""paper_2510_19608_b200 — B200-native exhaustive-search Kron reduction (Opti-KRON
hot path, reference `kronred::run_reduction`). See DESIGN.md."""
from .api import (  # noqa: F401
    Context, CudaError, Error, HostProblem, Network, ReducedModel, ReductionConfig, Result,
    ScenarioLibrary, SolverError, TraceRow, ValidationError, cdiv_selftest, enumerate_after,
    fp64_probe, lib, merge_best, nccl_unique_id, run_reduction, shard_range, validate,
)

__version__ = "0.1.0"
