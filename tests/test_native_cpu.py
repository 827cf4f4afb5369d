"""CPU-side checks of the boundary: the C-ABI library loads without a GPU,
exports every symbol include/cugenopt.h declares, NVRTC compiles user
operators for sm_100a (and rejects broken ones with a log), and the host
mirror of the reference API computes the same set-up values as the oracle."""

import ctypes as C
import math
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2603_19163_b200 as G
from oracle import aos as OA
from oracle import engine as OE
from oracle import problems as OP
from paper_2603_19163_b200 import _native as N
from paper_2603_19163_b200 import instances as I

ROOT = Path(__file__).resolve().parents[1]


def declared():
    text = (ROOT / "include" / "cugenopt.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(go_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = N.load(require_device=False)
    syms = declared()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(N.EXPORTED) == set(syms)
    assert lib.go_abi_version() == 1


def test_no_device_fails_loudly_without_cpu_fallback():
    lib = N.load(require_device=False)
    n = C.c_int(-1)
    if lib.go_device_count(C.byref(n)) == N.GO_OK and n.value > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(N.NativeUnavailable):
        N.load()
    prob = G.builtin_problem("tsp", G.InstanceData(distance_matrix=I.tsp_random(8, 1)))
    with pytest.raises(N.NativeUnavailable):
        G.run(prob, G.EngineConfig(population=2, team_size=4, max_generations=2))


def test_nvrtc_compiles_demo_operators(tmp_path, monkeypatch):
    monkeypatch.setenv("GO_JIT_CACHE", str(tmp_path))
    lib = N.load(require_device=False)
    ops = G.tsp_delta_operators()
    arr = (N.CustomOp * 3)(*[N.CustomOp(o.id, o.name.encode(), o.cuda.encode()) for o in ops])
    log = C.create_string_buffer(4096)
    key = C.create_string_buffer(65)
    assert lib.go_jit_compile(1, arr, 3, log, 4096, key) == N.GO_OK, log.value
    assert len(key.value) == 64
    assert list(tmp_path.glob("*.cubin"))
    bad = (N.CustomOp * 1)(N.CustomOp(110, b"broken_op", b"int x = ; ctx.swap(0, 1);"))
    assert lib.go_jit_compile(1, bad, 1, log, 4096, key) == N.GO_E_COMPILE
    assert b"broken_op" in log.value and b"error" in log.value


def test_registry_and_presets_match_oracle():
    for dist in (I.tsp_random(51, 51), I.tsp_lattice()[0]):
        prob = G.builtin_problem("tsp", G.InstanceData(distance_matrix=dist))
        cfg = prob.config()
        reg = G.build_registry(cfg, prob.device_sequences())
        G.apply_preset(reg, G.classify(cfg))
        oreg = OA.build_registry(OP.Tsp(dist).spec, None)  # the reference's full registry
        OA.apply_preset(oreg, OA.scale_of(OP.Tsp(dist).spec))
        assert reg.ids() == oreg.ids()
        assert reg.weights() == oreg.weights()
        assert reg.total() == sum(e.w for e in oreg.entries)


def test_population_sizing_rules():
    for hint, cache, ws, fast in [(108, 40 << 20, 763 << 10, 96 << 10), (80, 1, 10, 96 << 10),
                                  (148, 126 << 20, 781456, 227 << 10)]:
        assert G.adaptive_population_size(hint, cache, ws, fast) == \
            OE.population_size(hint, cache, ws, fast)
    # B200: one resident wave in the shared-memory path, L2 rule otherwise
    assert G.b200_population_size(148, 4, 126 << 20, 200_000, True) == 592
    assert G.b200_population_size(148, 4, 126 << 20, 50 << 20, False) == 2
    assert G.b200_population_size(148, 4, 126 << 20, 400_000, False) == 592


def test_host_init_matches_reference_draws():
    dist = I.tsp_random(20, 4)
    cfg = G.builtin_problem("tsp", G.InstanceData(distance_matrix=dist)).config()
    a = G.random_solution(cfg, G.engine.derived_rng(42, 2))
    b = OE.random_solution(OP.Tsp(dist).spec, OE.mt_stream(42, 2))
    assert a.row(0).tolist() == b.row(0).tolist()
    assert [p.tolist() for p in G.heuristic_candidates(dist)] == \
        [p.tolist() for p in OE.heuristic_perms(dist)]


def test_config_validation_mirrors_reference():
    with pytest.raises(ValueError):
        G.EngineConfig(team_size=0)
    with pytest.raises(ValueError):
        G.EngineConfig(cooling_alpha=0.0)
    with pytest.raises(ValueError):
        G.IslandsConfig(migration="star")
    with pytest.raises(ValueError):
        G.CustomOperator(100, "x", None, 0.0)
    with pytest.raises(ValueError):
        G.builtin_problem("nope", G.InstanceData())
    with pytest.raises(ValueError):
        G.builtin_problem("tsp", G.InstanceData(distance_matrix=np.array([[0, 1], [2, 0.0]])))
    assert math.isclose(sum(G.DEFAULT_K_WEIGHTS), 1.0)


def test_custom_problem_host_side():
    """CudaProblem (solve_custom) config / registry on the host; compile needs a device."""
    p = G.CudaProblem("integer", 12, "return 0.0;", lb=2, ub=5, maximize=True,
                      data={"w": np.arange(12.0)})
    cfg = p.config()
    assert (cfg.d1, cfg.d2, cfg.encoding.lower_bound, cfg.encoding.upper_bound) == (1, 12, 2, 5)
    reg = G.build_registry(cfg, p.device_sequences())
    assert reg.ids() == [7, 8, 13, 14, 15, 16]  # operators.py:597-615 for INTEGER
    assert p.payload_nbytes() == 96
    with pytest.raises(ValueError):
        G.CudaProblem("tree", 4, "return 0.0;")
    with pytest.raises(ValueError):
        G.CudaProblem("integer", 4, "return 0.0;")  # integer needs ub
    with pytest.raises(ValueError):
        G.solve_custom("binary", 4, n=5, compute_obj="return 0.0;")  # n must be 4


def test_result_record_schema_round_trip():
    """results.py:16-101: fixed key order, canonical text, strict parsing."""
    from paper_2603_19163_b200 import results as R
    rec = R.ResultRecord(problem="tsp", instance="lattice442", seed=42, objectives=[44200.0],
                         penalty=0.0, feasible=True, gap_pct=0.0, generations=16223,
                         elapsed_s=13.85, gens_per_sec=1171.3,
                         final_weights={"sequences": [], "k_steps": [0.8, 0.15, 0.05]},
                         profile={"scale": "large"}, config={"team_size": 128})
    text = R.emit_result(rec)
    assert list(json_keys(text)) == list(R.RESULT_SCHEMA_FIELDS)
    assert R.emit_result(R.parse_result(text)) == text
    assert R.parse_results(R.emit_results([rec, rec]))[1] == rec
    with pytest.raises(ValueError):
        R.ResultRecord.from_dict({"problem": "tsp"})
    assert "lattice442" in R.gap_table([rec])


def json_keys(text):
    import json
    return json.loads(text).keys()


def test_nondominated_sort_matches_oracle():
    """engine.py:370-420 (host, multi-objective init): product == oracle restatement."""
    from oracle import engine as OEng
    from paper_2603_19163_b200.core import Direction
    from paper_2603_19163_b200.engine import fast_nondominated_sort
    rng = np.random.default_rng(3)
    for trial in range(20):
        pts = rng.integers(0, 6, size=(int(rng.integers(1, 40)), 2)).astype(float)
        dirs = [Direction.MINIMIZE, Direction.MAXIMIZE if trial % 3 == 0 else Direction.MINIMIZE]
        odirs = ["maximize" if d is Direction.MAXIMIZE else "minimize" for d in dirs]
        assert fast_nondominated_sort(pts, dirs) == OEng.nondominated_sort(pts, odirs)
