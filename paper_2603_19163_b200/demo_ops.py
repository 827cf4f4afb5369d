"""Bundled user operators: delta-evaluation tour moves as CUDA snippets.

Device counterparts of the reference's `demo_ops.py:24-97` ("tsp-delta",
ids 100-102).  Each snippet is the body of
`template <class Ctx> __device__ void op(Ctx& ctx)` and is compiled by NVRTC
into the evolve kernel (paper §3.3.2).  They consume the lane stream in the
reference's draw order and evaluate the same float64 expressions, so the
move chosen for a given word stream is the reference's; the framework then
scores the resulting primitive move exactly (go_perm.cuh).

Ctx API: size(), at(p), dist(a, b), random(), randrange(lo, hi),
randbelow(n), swap(i, j), reverse(i, j), move_segment(start, len, pos),
insert(i, pos), relocate_best(start, len) (cooperative best-slot scan).
"""

from __future__ import annotations

from .operators import CustomOperator

PROBES = 24  # demo_ops.py:15

DELTA_TWO_OPT = r"""
  // demo_ops.py:24-45 — best of 24 sampled 2-opt moves, first improvement stops
  const int n = ctx.size();
  if (n < 4) return;
  bool have = false;
  double bd = 0.0;
  int bi = 0, bj = 0;
#pragma unroll 1
  for (int s = 0; s < 24; ++s) {
    const int i = ctx.randrange(0, n - 1);
    const int j = ctx.randrange(i + 1, n);
    if (i == 0 && j == n - 1) continue;
    const int a = ctx.at(i == 0 ? n - 1 : i - 1), b = ctx.at(i);
    const int c = ctx.at(j), d = ctx.at(j + 1 == n ? 0 : j + 1);
    const double delta = ctx.dist(a, c) + ctx.dist(b, d) - ctx.dist(a, b) - ctx.dist(c, d);
    if (!have || delta < bd) { have = true; bd = delta; bi = i; bj = j; }
    if (delta < -1e-12) break;
  }
  if (have) ctx.reverse(bi, bj);
"""

DELTA_OR_OPT = r"""
  // demo_ops.py:48-68 — relocate a 2-3 city strip to the best of 24 positions
  const int L = ctx.randrange(2, 4);
  const int n = ctx.size();
  if (n < L + 2) return;
  const int s = ctx.randbelow(n - L + 1);
  const int m = n - L;                       // rest[q] = tour[q < s ? q : q + L]
  const int f = ctx.at(s), l = ctx.at(s + L - 1);
  bool have = false;
  double bd = 0.0;
  int bp = 0;
#pragma unroll 1
  for (int t = 0; t < 24; ++t) {
    const int pos = ctx.randbelow(m + 1);
    const int qp = pos > 0 ? pos - 1 : m - 1, qn = pos == m ? 0 : pos;
    const int prev = ctx.at(qp < s ? qp : qp + L), nxt = ctx.at(qn < s ? qn : qn + L);
    const double delta = ctx.dist(prev, f) + ctx.dist(l, nxt) - ctx.dist(prev, nxt);
    if (!have || delta < bd) { have = true; bd = delta; bp = pos; }
  }
  ctx.move_segment(s, L, bp);
"""

DELTA_NODE_INSERT = r"""
  // demo_ops.py:71-89 — move one city to its best position over the whole tour.
  // The O(n) scan is handed to the framework (ctx.relocate_best): same float64
  // expression d(prev,c) + d(c,next) - d(prev,next), same first-minimum rule,
  // evaluated 32 slots at a time by a whole warp instead of one lane.
  const int n = ctx.size();
  if (n < 4) return;
  const int i = ctx.randbelow(n);
  ctx.relocate_best(i, 1);
"""

# The same operator written as a plain per-lane loop (kept for comparison and
# as an example of a self-contained snippet; selected by
# tsp_delta_operators(cooperative=False)).
DELTA_NODE_INSERT_LOOP = r"""
  const int n = ctx.size();
  if (n < 4) return;
  const int i = ctx.randbelow(n);
  const int city = ctx.at(i);
  const int m = n - 1;                       // rest[q] = tour[q < i ? q : q + 1]
  int prev = ctx.at(m - 1 < i ? m - 1 : m);  // rest[-1]
  double dpc = ctx.dist(prev, city);
  double bd = 0.0;
  int bp = -1;
  // slot m (pos % m == 0) repeats slot 0's delta and can never win the
  // strict '<' scan, so the reference's m + 1 slots reduce to m
#pragma unroll 4
  for (int pos = 0; pos < m; ++pos) {
    const int nxt = ctx.at(pos + (pos >= i));
    const double dcn = ctx.dist(city, nxt);
    const double delta = dpc + dcn - ctx.dist(prev, nxt);
    if (bp < 0 || delta < bd) { bd = delta; bp = pos; }
    prev = nxt;
    dpc = dcn;  // dist(prev', city) == dist(city, nxt): TSP matrices are symmetric
  }
  ctx.insert(i, bp);
"""


def tsp_delta_operators(cooperative: bool = True) -> tuple[CustomOperator, ...]:
    return (
        CustomOperator(100, "delta_two_opt", None, 1.0, DELTA_TWO_OPT),
        CustomOperator(101, "delta_or_opt", None, 1.0, DELTA_OR_OPT),
        CustomOperator(102, "delta_node_insert", None, 1.0,
                       DELTA_NODE_INSERT if cooperative else DELTA_NODE_INSERT_LOOP),
    )


DEMO_OPERATOR_SETS = {"tsp-delta": tsp_delta_operators}


def demo_operator_set(name: str) -> tuple[CustomOperator, ...]:
    try:
        return DEMO_OPERATOR_SETS[name]()
    except KeyError:
        raise ValueError(f"unknown operator set {name!r}; available: "
                         f"{', '.join(sorted(DEMO_OPERATOR_SETS))}") from None
