"""B200-native cuGenOpt evolve engine — drop-in for the reference `genopt`
package's search API (run / EngineConfig / builtin_problem / CustomOperator).

Python is the host mirror of the reference interface; the hot path is
`libcugenopt.so` (hand-written sm_100a CUDA, NVRTC for user operators).
There is no CPU fallback: device calls raise `NativeUnavailable` without a
GPU.
"""

__version__ = "0.1.0"

from ._native import NativeError, NativeUnavailable
from .aos import DEFAULT_K_WEIGHTS, AosConfig
from .core import (ComparisonMode, Direction, Encoding, EncodingKind, Lexicographic, ObjDef,
                   ProblemConfig, RowModeKind, Solution, StructuralError, ValidityReport,
                   Weighted, compare, scalarize, validate_solution)
from .demo_ops import demo_operator_set, tsp_delta_operators
from .engine import (DeviceRun, EngineConfig, EvolverState, IslandsConfig, RunResult,
                     adaptive_population_size, b200_population_size, heuristic_candidates,
                     initialize_population, random_solution, run, scalar_fitness)
from .operators import (CustomOperator, SequenceEntry, SequenceRegistry, build_registry,
                        lns_scope)
from .problems import (BUILTIN_NAMES, InstanceData, ProblemDefinition, builtin_problem,
                       evaluate)
from .profiles import PRESETS, ProblemProfile, Scale, WeightPreset, apply_preset, classify


def solve_tsp(dist_matrix, time_limit=30.0, **kw) -> RunResult:
    """PAPER.md:850-856 `cugenopt.solve_tsp(dist_matrix, time_limit=30)`."""
    cfg = EngineConfig(time_limit_seconds=time_limit,
                       max_generations=kw.pop("max_generations", 10 ** 9), **kw)
    return run(builtin_problem("tsp", InstanceData(distance_matrix=dist_matrix)), cfg)


__all__ = [name for name in dir() if not name.startswith("_")]
