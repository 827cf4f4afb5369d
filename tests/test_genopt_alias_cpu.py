"""The drop-in switch: `install_genopt_alias()` and the repo's `genopt/` shim
make `import genopt` (and its submodules, and `python -m genopt`) resolve to
this package; every name the reference exports is there (genopt/__init__.py:8-63)."""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

REFERENCE_EXPORTS = """DEFAULT_K_WEIGHTS AosConfig AosStats record sample_k sample_sequence
stagnation_check_and_reset update_weights BUILTIN_NAMES builtin_problem ComparisonMode Direction
Encoding EncodingKind Lexicographic ObjDef ProblemConfig RowModeKind Solution StructuralError
ValidityReport Weighted compare scalarize validate_solution EngineConfig EvolverState
IslandsConfig RunResult adaptive_population_size elite_inject evolve_generation
fast_nondominated_sort heuristic_candidates initialize_population island_migrate run DemoInstance
demo_instance demo_instances CustomOperator OperatorContext SequenceRegistry apply_sequence
build_registry lns_scope register_custom InstanceData ProblemDefinition evaluate PRESETS
ProblemProfile Scale WeightPreset apply_preset classify""".split()


def test_every_reference_export_is_present():
    import paper_2603_19163_b200 as G
    assert [n for n in REFERENCE_EXPORTS if not hasattr(G, n)] == []


def test_alias_and_submodules_in_a_fresh_interpreter():
    code = ("import paper_2603_19163_b200 as P; P.install_genopt_alias(); import genopt, "
            "genopt.engine, genopt.builtins, genopt.aos; "
            "assert genopt is P and genopt.engine.run is P.run; "
            "assert genopt.builtins.builtin_problem is P.builtin_problem; print('ok')")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=str(ROOT),
                       env=dict(os.environ, PYTHONPATH=str(ROOT)), timeout=120)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr


def test_python_dash_m_genopt_through_the_shim():
    r = subprocess.run([sys.executable, "-m", "genopt", "list-problems"], capture_output=True,
                       text=True, cwd="/tmp", env=dict(os.environ, PYTHONPATH=str(ROOT)),
                       timeout=120)
    assert r.returncode == 0 and "tsp" in r.stdout and "vrptw" in r.stdout, r.stderr
