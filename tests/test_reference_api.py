"""The reference's own test suite run against this package (drop-in check).

`tools/stage_reference.sh` copies the unmodified reference (package + its
tests and fixtures) under baseline/_ref/ — git-ignored, never committed, but
shipped with gpurun snapshots so the GPU box has it.  The plugin
tests/refapi/genopt_alias.py makes `import genopt` resolve to
paper_2603_19163_b200 before the reference's test modules are collected, and
the tests then run unchanged from the reference package directory (its
fixtures use relative paths).

* CPU (here): the host-only modules — core types, AOS helpers, profiles,
  parsers, population sizing, heuristic candidates, Pareto sorting.
* GPU: the API-level modules that drive the device — run(), evaluate(),
  initialisation, island helpers, evolve_generation, the CLI and result
  documents, the integration tests and the acceptance criteria — minus the
  deviations listed in DEVIATIONS (each one is a documented difference:
  MT19937 trajectories, Python-callback problems / operators).
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_PKG = ROOT / "baseline" / "_ref" / "reference_pkg"


def _staged() -> bool:
    if (REF_PKG / "tests").is_dir():
        return True
    if Path("/root/reference/pkg/tests").is_dir():  # build container: stage it
        r = subprocess.run(["sh", str(ROOT / "tools" / "stage_reference.sh")],
                           capture_output=True, text=True, timeout=600)
        return r.returncode == 0 and (REF_PKG / "tests").is_dir()
    return False


def _run(targets, deselect=(), timeout=1800):
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    cmd = [sys.executable, "-m", "pytest", "-p", "no:cacheprovider", "-p",
           "tests.refapi.genopt_alias", "-q", "-rf", *targets]
    for d in deselect:
        cmd += ["--deselect", d]
    return subprocess.run(cmd, cwd=str(REF_PKG), env=env, capture_output=True, text=True,
                          timeout=timeout)


HOST_ONLY = [
    "tests/test_aos.py", "tests/test_core.py", "tests/test_profiles.py", "tests/test_parsers.py",
    "tests/test_engine.py::TestHeuristicCandidates", "tests/test_engine.py::TestNonDominatedSort",
    "tests/test_engine.py::TestPopulationSizing",
]

DEVICE = ["tests/test_engine.py", "tests/test_integration.py", "tests/test_results_cli.py",
          "tests/test_problems.py", "tests/test_acceptance.py"]

# Known, documented deviations:
DEVIATIONS = [
    # MT19937 lane trajectory replayed with the reference's Python operators and
    # compared with evolve_generation's result: the device draws Philox words
    "tests/test_engine.py::TestEvolveGeneration::test_tie_breaks_to_lowest_lane",
    # problems defined by Python callbacks (ProblemDefinition subclasses): no
    # device path, by design (no CPU fallback); restated as CUDA snippets in
    # this repo's tests instead
    "tests/test_engine.py::TestInitializePopulation::test_multi_objective_keeps_first_front",
    # float-valued distances: a candidate whose tour is a re-ordering of the same
    # edges (whole-row operators) has a device length that can differ from the
    # current Φ by one ulp in either direction (different summation order), so
    # at T = 0 the exact numpy trajectory may rise by one ulp; integer-valued
    # instances are bit-exact
    "tests/test_engine.py::TestEvolveGeneration::test_zero_temperature_is_pure_hill_climbing",
    # (test_problem_seed_candidates_join_pool / test_invalid_seed_candidate_rejected subclass
    # the built-in TSP and override init_candidates only: they run on the device)
]


def test_reference_host_suite_against_package():
    if not _staged():
        pytest.skip("reference not staged (tools/stage_reference.sh)")
    r = _run(HOST_ONLY, timeout=600)
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout.splitlines()[-1]


@pytest.mark.gpu
def test_reference_device_suite_against_package():
    if not _staged():
        pytest.skip("reference not staged (tools/stage_reference.sh)")
    r = _run(DEVICE, DEVIATIONS)
    assert r.returncode == 0, r.stdout[-8000:] + r.stderr[-2000:]
