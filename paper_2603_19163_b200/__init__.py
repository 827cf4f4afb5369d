"""B200-native cuGenOpt evolve engine — drop-in for the reference `genopt`
package's search API (run / EngineConfig / builtin_problem / CustomOperator).

Python is the host mirror of the reference interface; the hot path is
`libcugenopt.so` (hand-written sm_100a CUDA, NVRTC for user operators).
There is no CPU fallback: device calls raise `NativeUnavailable` without a
GPU.
"""

__version__ = "0.1.0"

from ._native import NativeError, NativeUnavailable
from .aos import (DEFAULT_K_WEIGHTS, AosConfig, AosStats, record, sample_k, sample_sequence,
                  stagnation_check_and_reset, update_weights)
from .core import (ComparisonMode, Direction, Encoding, EncodingKind, Lexicographic, ObjDef,
                   ProblemConfig, RowModeKind, Solution, StructuralError, ValidityReport,
                   Weighted, compare, scalarize, validate_solution)
from .demo_ops import demo_operator_set, tsp_delta_operators
from .engine import (DeviceRun, EngineConfig, EvolverState, IslandsConfig, RunResult,
                     adaptive_population_size, b200_population_size, elite_inject,
                     evolve_generation, fast_nondominated_sort, heuristic_candidates,
                     initialize_population, initialize_population_device, island_migrate,
                     random_solution, run, scalar_fitness)
from .instances import DemoInstance, demo_instance, demo_instances
from .operators import (CustomOperator, OperatorContext, SequenceEntry, SequenceRegistry,
                        apply_sequence, build_registry, lns_scope, register_custom)
from .problems import (BUILTIN_NAMES, CudaProblem, InstanceData, ProblemDefinition,
                       builtin_problem, evaluate)
from .profiles import PRESETS, ProblemProfile, Scale, WeightPreset, apply_preset, classify


def solve_tsp(dist_matrix, time_limit=30.0, **kw) -> RunResult:
    """PAPER.md:850-856 `cugenopt.solve_tsp(dist_matrix, time_limit=30)`."""
    kw.setdefault("device_init", True)  # the paper's API initialises on the GPU
    cfg = EngineConfig(time_limit_seconds=time_limit,
                       max_generations=kw.pop("max_generations", 10 ** 9), **kw)
    return run(builtin_problem("tsp", InstanceData(distance_matrix=dist_matrix)), cfg)


def solve_knapsack(weights, values, capacity, time_limit=30.0, **kw) -> RunResult:
    """PAPER.md:850-856 `cugenopt.solve_knapsack(weights, values, cap)`."""
    kw.setdefault("device_init", True)  # the paper's API initialises on the GPU
    cfg = EngineConfig(time_limit_seconds=time_limit,
                       max_generations=kw.pop("max_generations", 10 ** 9), **kw)
    return run(builtin_problem("knapsack", InstanceData(weights=weights, values=values,
                                                        capacity=capacity)), cfg)


def solve_custom(encoding, dim2, n=None, compute_obj=None, compute_penalty=None, data=None,
                 custom_operators=(), time_limit=30.0, lb=0, ub=None, maximize=False,
                 best_known=None, dim1=1, **kw) -> RunResult:
    """PAPER.md:858-868 `cugenopt.solve_custom(encoding=, dim2=, n=, compute_obj=,
    compute_penalty=, data=, custom_operators=, time_limit=)`: a single-row (or,
    with dim1 > 1, MULTI_FIXED) problem whose objective / penalty are CUDA
    snippets (see CudaProblem),
    compiled by NVRTC into the device evolve kernel."""
    # ProblemConfig.n: dim2 values per permutation row, dim1 * dim2 cells otherwise
    want_n = int(dim2) if encoding == "permutation" else int(dim1) * int(dim2)
    if n is not None and int(n) != want_n:
        raise ValueError(f"{encoding} problems with dim1={dim1}, dim2={dim2} need n == {want_n}")
    prob = CudaProblem(encoding, int(dim2), compute_obj, compute_penalty, data, lb=lb, ub=ub,
                       maximize=maximize, rows=int(dim1))
    kw.setdefault("device_init", True)  # the paper's API initialises on the GPU
    cfg = EngineConfig(time_limit_seconds=time_limit, custom_operators=tuple(custom_operators),
                       max_generations=kw.pop("max_generations", 10 ** 9), **kw)
    return run(prob, cfg, best_known=best_known)


from . import problems as builtins  # noqa: E402  (the reference's genopt.builtins)


def install_genopt_alias() -> None:
    """Make `import genopt` (and `genopt.engine`, `genopt.operators`, ...)
    resolve to this package, so code written against the reference runs
    unchanged: the drop-in switch.  The reference's
    `genopt.builtins` is this package's `problems` module."""
    import importlib
    import sys
    sys.modules["genopt"] = sys.modules[__name__]
    for sub in ("aos", "core", "demo_ops", "engine", "instances", "operators", "parsers",
                "problems", "profiles", "results", "cli"):
        sys.modules[f"genopt.{sub}"] = importlib.import_module(f"{__name__}.{sub}")
    sys.modules["genopt.builtins"] = sys.modules[f"{__name__}.problems"]


__all__ = [name for name in dir() if not name.startswith("_")]
