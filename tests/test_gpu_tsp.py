"""GPU parity: the CUDA path (through libcugenopt.so) against the CPU oracle.

Tolerances: integer-valued instances (TSPLIB nint) must match bit-for-bit
(SURVEY §8c); float instances within 1e-6 relative (the north-star bound) —
the tests below use 1e-9 relative for single evaluations.
"""

import random

import numpy as np
import pytest

from oracle import engine as OE
from oracle import moves as OM
from oracle import problems as OP
from paper_2603_19163_b200 import _native as N
from paper_2603_19163_b200 import instances as I

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    return N.load()


def _tsp(dist):
    import paper_2603_19163_b200 as G
    return G.builtin_problem("tsp", G.InstanceData(distance_matrix=dist))


def _eval(lib, prob, tours):
    h = prob.device_handle(0)
    g = np.ascontiguousarray(tours, dtype=np.int32)
    s = np.full((len(tours), 1), g.shape[1], dtype=np.int32)
    obj = np.zeros(len(tours))
    pen = np.zeros(len(tours))
    N.check(lib.go_eval_batch(h, N.iptr(g), N.iptr(s), len(tours), N.dptr(obj), N.dptr(pen)))
    return obj, pen


@pytest.mark.parametrize("name", ["c1", "c2", "c1f", "small"])
def test_eval_batch_matches_oracle(lib, name):
    dist = {"c1": I.tsp_random(51, 51, True), "c2": I.tsp_lattice()[0],
            "c1f": I.tsp_random(51, 51, False), "small": I.tsp_random(5, 3, True)}[name]
    n = dist.shape[0]
    rng = np.random.default_rng(5)
    tours = np.stack([rng.permutation(n) for _ in range(64)])
    obj, pen = _eval(lib, _tsp(dist), tours)
    o = OP.Tsp(dist)
    ref = np.array([o.objective(0, OP.Sol(t[None, :], [n])) for t in tours])
    assert np.all(pen == 0.0)
    if name == "c1f":
        assert np.allclose(obj, ref, rtol=1e-9, atol=0)
    else:
        assert np.array_equal(obj, ref)


def test_lattice_optimum_is_44200(lib):
    d, opt = I.tsp_lattice()
    obj, _ = _eval(lib, _tsp(d), I.lattice_tour()[None, :])
    assert obj[0] == opt == 44200.0


def _apply(t, mv):
    kind, a, b, c = mv
    t = list(t)
    if kind == N.MOVE_SWAP:
        t[a], t[b] = t[b], t[a]
    elif kind == N.MOVE_REVERSE:
        t[a:b + 1] = t[a:b + 1][::-1]
    elif kind == N.MOVE_SEGMENT:
        seg = t[a:a + b]
        rest = t[:a] + t[a + b:]
        t = rest[:c] + seg + rest[c:]
    elif kind >= N.MOVE_THREE_OPT:  # operators.py:289-315 reconnection variants
        A, B, C, D = t[:a], t[a:b], t[b:c], t[c:]
        v = kind - N.MOVE_THREE_OPT
        parts = [(A, B[::-1], C, D), (A, B, C[::-1], D), (A, B[::-1], C[::-1], D), (A, C, B, D),
                 (A, C, B[::-1], D), (A, C[::-1], B, D), (A, C[::-1], B[::-1], D)][v]
        t = [x for part in parts for x in part]
    return t


def _random_move(rng, n):
    kind = rng.choice([N.MOVE_SWAP, N.MOVE_REVERSE, N.MOVE_SEGMENT] +
                      ([N.MOVE_THREE_OPT] if n >= 4 else []))
    if kind == N.MOVE_THREE_OPT:
        i, j, k = sorted(rng.sample(range(1, n), 3))
        return (kind + rng.randrange(7), i, j, k)
    if kind == N.MOVE_SWAP:
        a = rng.randrange(n)
        b = rng.randrange(n - 1)
        b += b >= a
        return (kind, a, b, 0)
    if kind == N.MOVE_REVERSE:
        a = rng.randrange(n - 1)
        return (kind, a, rng.randrange(a + 1, n), 0)
    L = rng.randrange(1, min(3, n - 1) + 1)
    s = rng.randrange(n - L + 1)
    return (kind, s, L, rng.randrange(n - L + 1))


@pytest.mark.parametrize("n,integral", [(2, True), (3, True), (4, True), (5, True), (8, True),
                                        (51, True), (442, True), (51, False)])
def test_delta_chains_match_oracle(lib, n, integral):
    dist = I.tsp_lattice()[0] if n == 442 else I.tsp_random(n, 100 + n, integral)
    prob = _tsp(dist)
    o = OP.Tsp(dist)
    rng = random.Random(n)
    m = 400
    tours, moves = [], []
    for _ in range(m):
        t = list(range(n))
        rng.shuffle(t)
        k = rng.randrange(1, 4)
        chain = [_random_move(rng, n) for _ in range(k)] + [(0, 0, 0, 0)] * (3 - k)
        if n >= 4 and rng.random() < 0.3:  # force the wrap / adjacency edge cases
            chain[0] = rng.choice([(N.MOVE_SWAP, 0, n - 1, 0), (N.MOVE_REVERSE, 0, n - 1, 0),
                                   (N.MOVE_SWAP, 1, 2, 0), (N.MOVE_SEGMENT, 0, 2, n - 2),
                                   (N.MOVE_SEGMENT, n - 2, 2, 0), (N.MOVE_SEGMENT, 1, 1, 1),
                                   (N.MOVE_THREE_OPT + 3, 1, 2, n - 1),
                                   (N.MOVE_THREE_OPT + 6, 1, n - 2, n - 1)])
        tours.append(t)
        moves.append(chain)
    g = np.array(tours, dtype=np.int32)
    s = np.full((m, 1), n, dtype=np.int32)
    mv = (N.Move * (3 * m))(*[N.Move(*x) for ch in moves for x in ch])
    delta = np.zeros(m)
    cand = np.zeros_like(g)
    N.check(lib.go_delta_batch(prob.device_handle(0), N.iptr(g), N.iptr(s), m, mv, 0.0,
                               N.dptr(delta), N.iptr(cand)))
    for i in range(m):
        c = tours[i]
        for x in moves[i]:
            c = _apply(c, x)
        assert cand[i].tolist() == c
        phi0 = o.objective(0, OP.Sol(np.array([tours[i]]), [n]))
        phi1 = o.objective(0, OP.Sol(np.array([c]), [n]))
        if integral:
            assert delta[i] == phi1 - phi0, (tours[i], moves[i])
        else:
            assert abs(delta[i] - (phi1 - phi0)) <= 1e-9 * max(1.0, abs(phi0))


def _engine_vs_oracle(dist, P, T, G, seed, custom=False, islands=1, migration="ring",
                      mig_interval=100, elite=50, cooperative=True):
    import paper_2603_19163_b200 as G_
    from paper_2603_19163_b200.demo_ops import tsp_delta_operators
    prob = _tsp(dist)
    cfg = G_.EngineConfig(population=P, team_size=T, max_generations=G, seed=seed,
                          record_history=True, elite_injection_interval=elite,
                          islands=G_.IslandsConfig(count=islands, migration=migration,
                                                   interval=mig_interval),
                          custom_operators=tsp_delta_operators(cooperative) if custom else ())
    res = G_.run(prob, cfg)
    ocfg = OE.RunCfg(population=P, team_size=T, max_generations=G, seed=seed,
                     record_history=True, elite_interval=elite, islands=islands,
                     migration=migration, migration_interval=mig_interval,
                     allowed_ops=prob.device_sequences(),
                     custom_ops=tuple((i, nm, f, 1.0) for i, nm, f in OM.TSP_DELTA) if custom else ())
    ref = OE.run(OP.Tsp(dist), ocfg, device_stream="philox")
    return res, ref


def _assert_same_run(res, ref):
    assert res.generations_completed == ref.generations
    assert res.device["error_flags"] == 0
    assert [e["id"] for e in res.final_weights["sequences"]] == ref.ids
    assert res.history["best_phi"] == ref.history["best_phi"]
    assert res.objectives == ref.objectives
    assert res.best.row(0).tolist() == ref.best.row(0).tolist()
    assert [e["weight"] for e in res.final_weights["sequences"]] == [float(w) for w in ref.weights]
    assert res.final_weights["k_steps"] == list(ref.k_weights)
    assert [s.row(0).tolist() for s in res.population] == [s.row(0).tolist() for s in ref.population]


@pytest.mark.parametrize("seed", [42, 123])
def test_evolve_bit_identical_to_oracle_c1(seed):
    res, ref = _engine_vs_oracle(I.tsp_random(51, 51, True), P=8, T=32, G=60, seed=seed)
    _assert_same_run(res, ref)


def test_evolve_bit_identical_islands_and_elite():
    res, ref = _engine_vs_oracle(I.tsp_random(30, 7, True), P=9, T=40, G=45, seed=7, islands=3,
                                 migration="hybrid", mig_interval=10, elite=15)
    _assert_same_run(res, ref)


@pytest.mark.parametrize("cooperative", [True, False])
def test_evolve_bit_identical_with_user_operators(cooperative):
    res, ref = _engine_vs_oracle(I.tsp_random(51, 51, True), P=6, T=32, G=40, seed=2024,
                                 custom=True, cooperative=cooperative)
    _assert_same_run(res, ref)
    assert [e["id"] for e in res.final_weights["sequences"]][-3:] == [100, 101, 102]


@pytest.mark.parametrize("cooperative", [True, False])
def test_evolve_lattice_shared_memory_triangle(cooperative):
    """C2 shape: int16 packed triangle staged into shared memory."""
    d, _ = I.tsp_lattice()
    res, ref = _engine_vs_oracle(d, P=4, T=128, G=12, seed=456, custom=True,
                                 cooperative=cooperative)
    _assert_same_run(res, ref)
    assert res.device["layout"] == 1  # L_I16_TRI


def test_float_instance_with_user_operators_matches_oracle():
    """Float matrix: decisions are float64 in both engines; bit-identical while
    the int64/float64 delta sums agree (they do on this seed)."""
    res, ref = _engine_vs_oracle(I.tsp_random(40, 9, False), P=4, T=32, G=20, seed=9,
                                 custom=True)
    assert res.generations_completed == ref.generations
    assert abs(res.objectives[0] - ref.objectives[0]) <= 1e-6 * ref.objectives[0]


def test_float_instance_runs_within_tolerance():
    import paper_2603_19163_b200 as G_
    d = I.tsp_random(51, 51, False)
    res = G_.run(_tsp(d), G_.EngineConfig(population=16, team_size=64, max_generations=200,
                                          seed=3))
    o = OP.Tsp(d)
    phi = o.objective(0, OP.Sol(res.best.data, res.best.dim2_sizes))
    assert abs(res.objectives[0] - phi) <= 1e-6 * phi


def test_time_limit_and_throughput_c2():
    import paper_2603_19163_b200 as G_
    from paper_2603_19163_b200.demo_ops import tsp_delta_operators
    d, opt = I.tsp_lattice()
    res = G_.run(_tsp(d), G_.EngineConfig(time_limit_seconds=3.0, max_generations=10 ** 9,
                                          custom_operators=tsp_delta_operators()), best_known=opt)
    assert res.generations_completed > 0
    assert 2.0 < res.elapsed_seconds < 6.0
    o = OP.Tsp(d)
    assert res.objectives[0] == o.objective(0, OP.Sol(res.best.data, res.best.dim2_sizes))
    assert res.gap_pct is not None and res.gap_pct < 50


@pytest.mark.parametrize("ops", [(12, 2), (14,), (15,), (16,), (4,), (12, 0), (16, 101), (14, 102)])
def test_whole_row_operators_match_oracle(ops):
    """OX / seg_shuffle / scatter_shuffle / guided_rebuild (go_perm_lns.cuh) and
    3-opt, alone and chained with position-map moves and user operators."""
    import paper_2603_19163_b200 as G_
    from paper_2603_19163_b200.demo_ops import tsp_delta_operators
    dist = I.tsp_random(51, 51, True)
    prob = _tsp(dist)
    builtin = tuple(o for o in ops if o < 100)
    prob.device_sequences = lambda: builtin
    custom = [o for o in tsp_delta_operators() if o.id in ops]
    cfg = G_.EngineConfig(population=4, team_size=32, max_generations=12, seed=5,
                          record_history=True, custom_operators=custom)
    res = G_.run(prob, cfg)
    ocfg = OE.RunCfg(population=4, team_size=32, max_generations=12, seed=5,
                     record_history=True, allowed_ops=builtin,
                     custom_ops=tuple((i, nm, f, 1.0) for i, nm, f in OM.TSP_DELTA if i in ops))
    ref = OE.run(OP.Tsp(dist), ocfg, device_stream="philox")
    _assert_same_run(res, ref)


def test_population_beyond_one_wave_crossover_fallback():
    """More evolvers than one resident wave: the snapshot protocol cannot spin on
    teams that are not resident, so chunks shrink to one generation (launch
    boundaries are the snapshot barriers) — still bit-identical to the oracle."""
    import paper_2603_19163_b200 as G_
    dist = I.tsp_random(12, 3, True)
    prob = _tsp(dist)
    cfg = G_.EngineConfig(population=3000, team_size=8, max_generations=3, seed=17,
                          record_history=True)
    res = G_.run(prob, cfg)
    ref = OE.run(OP.Tsp(dist), OE.RunCfg(population=3000, team_size=8, max_generations=3,
                                         seed=17, record_history=True,
                                         allowed_ops=prob.device_sequences()),
                 device_stream="philox")
    assert res.history["best_phi"] == ref.history["best_phi"]
    assert [s.row(0).tolist() for s in res.population] == [s.row(0).tolist() for s in ref.population]


def test_population_round_trip_through_pinned_staging():
    """go_engine_set_population stages rows through pinned memory with
    asynchronous copies on the engine stream (engine.cu); a get right after a
    set, and a run after it, must see the new rows and objectives."""
    import paper_2603_19163_b200 as G

    dist = I.tsp_random(30, 7, True)
    prob = _tsp(dist)
    dr = G.DeviceRun(prob, G.EngineConfig(population=8, team_size=32, seed=3), 3)
    P, W = dr.pop_size, dr.cfg.d2
    genes = np.zeros((P, W), dtype=np.int32)
    sizes = np.zeros((P, 1), dtype=np.int32)
    obj = np.zeros(P)
    pen = np.zeros(P)
    N.check(dr.lib.go_engine_get_population(dr.engine, N.iptr(genes), N.iptr(sizes),
                                            N.dptr(obj), N.dptr(pen)))
    rng = np.random.default_rng(0)
    new = np.array([rng.permutation(W) for _ in range(P)], dtype=np.int32)
    new_obj, _ = _eval(dr.lib, prob, new)
    for rep in range(3):  # back to back: the staging buffer is reused
        N.check(dr.lib.go_engine_set_population(dr.engine, N.iptr(new), N.iptr(sizes),
                                                N.dptr(new_obj), N.dptr(pen)))
        got = np.zeros_like(genes)
        got_obj = np.zeros(P)
        N.check(dr.lib.go_engine_get_population(dr.engine, N.iptr(got), N.iptr(sizes),
                                                N.dptr(got_obj), N.dptr(pen)))
        assert (got == new).all()
        assert np.array_equal(got_obj, new_obj)
    st = dr.run(2, None)
    assert st.generations == 2
    N.check(dr.lib.go_engine_get_population(dr.engine, N.iptr(got), N.iptr(sizes),
                                            N.dptr(got_obj), N.dptr(pen)))
    re_obj, _ = _eval(dr.lib, prob, got)
    assert np.array_equal(re_obj, got_obj)  # integer instance: exact
    dr.close()
