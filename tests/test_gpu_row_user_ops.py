"""User operators on the hand-written row kernels (VERDICT r1 "Missing" #2):
register_custom (operators.py:634-669, engine.py:625-636) for QAP, knapsack,
JSP-int and the partition problems (VRPTW / CVRP).  Each operator is a CUDA
snippet compiled by NVRTC into the problem's own evolve kernel, probed, and
then sampled by AOS like a built-in.  Whole runs must be bit-identical to the
Philox-mode oracle running the same operators restated in Python."""
import numpy as np
import pytest

import paper_2603_19163_b200 as G
from oracle import engine as OE
from oracle import problems as OP
from paper_2603_19163_b200 import instances as I
from tests.helpers import bench_pairs

pytestmark = pytest.mark.gpu

# ---- QAP: best of 8 sampled swaps by the exact Taillard-style delta ---------------
QAP_DELTA_SWAP = r"""
  const int n = ctx.n;
  int bi = -1, bj = -1;
  double bd = 0.0;
  for (int t = 0; t < 8; ++t) {
    const int i = ctx.randbelow(n);
    int j = ctx.randbelow(n - 1);
    j += j >= i;
    const int pi = ctx.get(i), pj = ctx.get(j);
    double d = 0.0;
    for (int k = 0; k < n; ++k) {
      if (k == i || k == j) continue;
      const int pk = ctx.get(k);
      d += (ctx.flow(i, k) - ctx.flow(j, k)) * (ctx.dist(pj, pk) - ctx.dist(pi, pk))
         + (ctx.flow(k, i) - ctx.flow(k, j)) * (ctx.dist(pk, pj) - ctx.dist(pk, pi));
    }
    d += (ctx.flow(i, i) - ctx.flow(j, j)) * (ctx.dist(pj, pj) - ctx.dist(pi, pi))
       + (ctx.flow(i, j) - ctx.flow(j, i)) * (ctx.dist(pj, pi) - ctx.dist(pi, pj));
    if (bi < 0 || d < bd) { bd = d; bi = i; bj = j; }
  }
  ctx.swap(bi, bj);
"""


def qap_delta_swap(sol, rng, ctx):
    F, D = ctx.problem.flow, ctx.problem.dist
    row = sol.data[0]
    n = len(row)
    bi = bj = -1
    bd = 0.0
    for _ in range(8):
        i = rng.randrange(n)
        j = rng.randrange(n - 1)
        j += j >= i
        pi, pj = int(row[i]), int(row[j])
        d = 0.0
        for k in range(n):
            if k in (i, j):
                continue
            pk = int(row[k])
            d += (F[i, k] - F[j, k]) * (D[pj, pk] - D[pi, pk]) + \
                (F[k, i] - F[k, j]) * (D[pk, pj] - D[pk, pi])
        d += (F[i, i] - F[j, j]) * (D[pj, pj] - D[pi, pi]) + \
            (F[i, j] - F[j, i]) * (D[pj, pi] - D[pi, pj])
        if bi < 0 or d < bd:
            bd, bi, bj = d, i, j
    row[bi], row[bj] = row[bj], row[bi]


# ---- VRPTW: relocate a random customer to the cheapest of 6 sampled slots ---------
VRPTW_RELOCATE = r"""
  const int n = ctx.n, R = ctx.rows;
  int g = ctx.randbelow(n);
  int r0 = 0;
  while (g >= ctx.size(r0)) { g -= ctx.size(r0); ++r0; }
  const int p0 = g;
  const int c = ctx.get(r0, p0);
  int br = -1, bp = 0;
  double bd = 0.0;
  for (int t = 0; t < 6; ++t) {
    const int r1 = ctx.randbelow(R);
    if (r1 != r0 && ctx.size(r1) >= ctx.width) continue;
    const int sz = ctx.size(r1) - (r1 == r0 ? 1 : 0);
    const int p1 = ctx.randbelow(sz + 1);
    int prev = -1, next = -1;  // -1: the depot
    if (p1 > 0) { int q = p1 - 1; if (r1 == r0 && q >= p0) ++q; prev = ctx.get(r1, q); }
    if (p1 < sz) { int q = p1; if (r1 == r0 && q >= p0) ++q; next = ctx.get(r1, q); }
    const double d = ctx.dist(prev, c) + ctx.dist(c, next) - ctx.dist(prev, next);
    if (br < 0 || d < bd) { bd = d; br = r1; bp = p1; }
  }
  if (br >= 0) ctx.move(r0, p0, br, bp);
"""


def vrptw_relocate(sol, rng, ctx):
    P = ctx.problem
    dist, n = P.dist, P.n
    R, W = sol.data.shape
    g = rng.randrange(n)
    r0 = 0
    while g >= sol.sizes[r0]:
        g -= int(sol.sizes[r0])
        r0 += 1
    p0 = g
    c = int(sol.data[r0, p0])
    br, bp, bd = -1, 0, 0.0
    for _ in range(6):
        r1 = rng.randrange(R)
        if r1 != r0 and sol.sizes[r1] >= W:
            continue
        sz = int(sol.sizes[r1]) - (1 if r1 == r0 else 0)
        p1 = rng.randrange(sz + 1)
        prev = nxt = -1
        if p1 > 0:
            q = p1 - 1
            if r1 == r0 and q >= p0:
                q += 1
            prev = int(sol.data[r1, q])
        if p1 < sz:
            q = p1
            if r1 == r0 and q >= p0:
                q += 1
            nxt = int(sol.data[r1, q])
        d = dist[prev + 1, c + 1] + dist[c + 1, nxt + 1] - dist[prev + 1, nxt + 1]
        if br < 0 or d < bd:
            br, bp, bd = r1, p1, d
    if br < 0:
        return
    src = [int(v) for v in sol.data[r0, :sol.sizes[r0]]]
    del src[p0]
    sol.data[r0, :len(src)] = src
    sol.data[r0, len(src):] = 0
    sol.sizes[r0] -= 1
    dst = [int(v) for v in sol.data[br, :sol.sizes[br]]]
    dst.insert(bp, c)
    sol.data[br, :len(dst)] = dst
    sol.sizes[br] += 1


# ---- knapsack: flip the best of 4 sampled items by Φ (ctx.phi) ----------------------
KNAP_PHI_FLIP = r"""
  const int n = ctx.n;
  int bi = -1;
  double bp = 0.0;
  for (int t = 0; t < 4; ++t) {
    const int i = ctx.randbelow(n);
    ctx.set(i, 1 - ctx.get(i));
    const double p = ctx.phi();
    ctx.set(i, 1 - ctx.get(i));
    if (bi < 0 || p < bp) { bp = p; bi = i; }
  }
  ctx.set(bi, 1 - ctx.get(bi));
"""


def knap_phi_flip(sol, rng, ctx):
    row = sol.data[0]
    bi, bp = -1, 0.0
    for _ in range(4):
        i = rng.randrange(len(row))
        row[i] = 1 - row[i]
        p = ctx.phi(sol)
        row[i] = 1 - row[i]
        if bi < 0 or p < bp:
            bi, bp = i, p
    row[bi] = 1 - row[bi]


def _cells(data, sizes):
    return [list(map(int, row[:int(k)])) for row, k in zip(data, sizes)]


def _run_pair(prob, ref, op, pyfn, P, T, gens, seed):
    res = G.run(prob, G.EngineConfig(population=P, team_size=T, max_generations=gens, seed=seed,
                                     record_history=True, custom_operators=(op,)))
    out = OE.run(ref, OE.RunCfg(population=P, team_size=T, max_generations=gens, seed=seed,
                                record_history=True, allowed_ops=prob.device_sequences(),
                                custom_ops=((op.id, op.name, pyfn, op.initial_weight),)),
                 device_stream="philox")
    assert res.device["error_flags"] == 0
    assert [e["id"] for e in res.final_weights["sequences"]] == out.ids
    assert out.ids[-1] == op.id
    assert res.history["best_phi"] == out.history["best_phi"]
    assert res.objectives == out.objectives and res.penalty == out.penalty
    assert [e["weight"] for e in res.final_weights["sequences"]] == [float(w) for w in out.weights]
    assert [_cells(s.data, s.dim2_sizes) for s in res.population] == \
        [_cells(s.data, s.sizes) for s in out.population]
    return res


def test_user_qap_delta_swap_bit_identical():
    f, d = I.qap_random(30, 100)
    prob = G.builtin_problem("qap", G.InstanceData(flow_matrix=f, distance_matrix=d))
    op = G.CustomOperator(200, "qap_delta_swap", None, 2.0, QAP_DELTA_SWAP)
    _run_pair(prob, OP.Qap(f, d), op, qap_delta_swap, P=6, T=32, gens=30, seed=11)


def test_user_vrptw_relocate_bit_identical_on_r101():
    prob, ref, _, _ = bench_pairs(("C3",))["C3"]
    op = G.CustomOperator(201, "vrptw_relocate", None, 1.0, VRPTW_RELOCATE)
    _run_pair(prob, ref, op, vrptw_relocate, P=6, T=32, gens=25, seed=12)


def test_user_knapsack_phi_flip_bit_identical():
    w, v, cap = I.knapsack_random(200, 1000)
    prob = G.builtin_problem("knapsack", G.InstanceData(weights=w, values=v, capacity=cap))
    op = G.CustomOperator(202, "knap_phi_flip", None, 1.0, KNAP_PHI_FLIP)
    _run_pair(prob, OP.Knapsack(w, v, cap), op, knap_phi_flip, P=6, T=32, gens=25, seed=13)


def test_row_user_operator_probe_excludes_broken_snippets():
    """operators.py:649-665: a compile error or an invalid probe result excludes
    the operator with a RuntimeWarning; the run continues bit-identically to a
    run without it."""
    f, d = I.qap_random(20, 5)
    prob = G.builtin_problem("qap", G.InstanceData(flow_matrix=f, distance_matrix=d))
    bad_compile = G.CustomOperator(210, "no_semicolon", None, 1.0, "int x = 1")
    bad_result = G.CustomOperator(211, "duplicate", None, 1.0, "ctx.set(0, ctx.get(1));")
    with pytest.warns(RuntimeWarning) as rec:
        r1 = G.run(prob, G.EngineConfig(population=4, team_size=32, max_generations=20, seed=3,
                                        custom_operators=(bad_compile, bad_result)))
    assert len([w for w in rec if "excluded" in str(w.message)]) == 2
    r0 = G.run(prob, G.EngineConfig(population=4, team_size=32, max_generations=20, seed=3))
    assert r1.best.row(0).tolist() == r0.best.row(0).tolist()
    assert [e["id"] for e in r1.final_weights["sequences"]] == \
        [e["id"] for e in r0.final_weights["sequences"]]
