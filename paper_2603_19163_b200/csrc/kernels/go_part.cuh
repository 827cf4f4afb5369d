// go_part.cuh — partition-encoding (VRPTW / CVRP) operators and evaluation.
//
// Compact lane row: cells[0..n) = the routes concatenated in row order, then
// sizes[0..d1) (the reference's d1 x d2 matrix + dim2_sizes, core.py:154-200,
// without the padding).  Global cell index g is exactly _nth_cell's order
// (operators.py:154-162).  Every operator is a port of the reference's
// MULTI_PARTITION branch with its draw order (operators.py:205-406, :468-499).
// Evaluation restates builtins.py:119-187 in the reference's arithmetic order:
// numpy pairwise sums for the edge / demand sums, Python's compensated sum()
// over route lengths, sequential capacity and lateness accumulation.
#pragma once
#include "go_common.cuh"
#include "go_row.cuh"

namespace go {

struct PartView {  // instance (float64 arrays, customer c at matrix index c + 1)
  const double* dist;  // (n+1) x (n+1)
  const double* demand;
  const double* ready;
  const double* due;
  const double* service;
  int n, d1, d2;
  double cap;
  int tw;  // 1: VRPTW (lateness), 0: CVRP
  int variant;         // 0 plain, 1 vrp_priority (precedence penalty), 2 vrp_nonlinear
  const double* prio;  // vrp_priority: priority per customer
};

struct PartCtx {
  Stream rng;  // by value (see RowCtx)
  short* cells;  // [n]
  short* sz;     // [d1]
  int n, d1, d2, n_cfg;
  int total;     // cells currently stored (n except inside an op)
  int err;
  const MateSel* mates;  // crossover mates (engine.py:553-559); rows = cells + sizes
  __device__ __forceinline__ int randbelow(int m) { return rng.randbelow(m); }
  __device__ __forceinline__ int randrange(int lo, int hi) { return rng.randrange(lo, hi); }
  __device__ __forceinline__ int start(int r) const {
    int s = 0;
#pragma unroll 1
    for (int q = 0; q < r; ++q) s += sz[q];
    return s;
  }
  __device__ __forceinline__ void cell_at(int g, int& r, int& p) const {
#pragma unroll 1
    for (int q = 0; q < d1; ++q) {
      if (g < sz[q]) {
        r = q;
        p = g;
        return;
      }
      g -= sz[q];
    }
    r = d1 - 1;
    p = 0;
  }
  __device__ __forceinline__ short remove(int r, int p) {
    const int gi = start(r) + p;
    const short v = cells[gi];
    for (int q = gi; q < total - 1; ++q) cells[q] = cells[q + 1];
    --total;
    sz[r] -= 1;
    return v;
  }
  __device__ __forceinline__ void insert(int r, int p, short v) {
    const int gi = start(r) + p;
    for (int q = total; q > gi; --q) cells[q] = cells[q - 1];
    cells[gi] = v;
    ++total;
    sz[r] += 1;
  }
  // _pick_row: rows with size >= min_size, uniform (operators.py:140-144)
  __device__ __forceinline__ int pick_row(int min_size) {
    int cnt = 0;
#pragma unroll 1
    for (int q = 0; q < d1; ++q) cnt += sz[q] >= min_size;
    if (cnt == 0) return -1;
    int k = randbelow(cnt);
#pragma unroll 1
    for (int q = 0; q < d1; ++q)
      if (sz[q] >= min_size && k-- == 0) return q;
    return -1;
  }
};

__device__ __forceinline__ void rev_short(short* a, int i, int j) {  // [i, j]
  while (i < j) {
    const short t = a[i];
    a[i] = a[j];
    a[j] = t;
    ++i;
    --j;
  }
}

// move block [a, a+L) so that it starts at b in the array without the block
__device__ __forceinline__ void move_block(short* c, int a, int L, int b) {
  if (L <= 0 || a == b) return;
  if (b > a) {  // range [a, b+L): rotate left by L
    rev_short(c, a, a + L - 1);
    rev_short(c, a + L, b + L - 1);
    rev_short(c, a, b + L - 1);
  } else {      // range [b, a+L): rotate right by L
    rev_short(c, b, a - 1);
    rev_short(c, a, a + L - 1);
    rev_short(c, b, a + L - 1);
  }
}

__device__ __forceinline__ void pop_swap(PartCtx& c) {
  const int total = c.total;
  if (total < 2) return;
  const int g1 = c.randbelow(total);
  int g2 = c.randbelow(total - 1);
  g2 += g2 >= g1;
  const short t = c.cells[g1];
  c.cells[g1] = c.cells[g2];
  c.cells[g2] = t;
}

__device__ __forceinline__ void pop_insert(PartCtx& c) {
  if (c.total == 0) return;
  int r1, p1;
  c.cell_at(c.randbelow(c.total), r1, p1);
  int cnt = 0;
  for (int r = 0; r < c.d1; ++r)
    cnt += (r == r1 && c.sz[r1] >= 2) || (r != r1 && c.sz[r] < c.d2);
  if (cnt == 0) return;
  int k = c.randbelow(cnt), r2 = -1;
  for (int r = 0; r < c.d1; ++r)
    if (((r == r1 && c.sz[r1] >= 2) || (r != r1 && c.sz[r] < c.d2)) && k-- == 0) {
      r2 = r;
      break;
    }
  const short v = c.remove(r1, p1);
  const int pos = c.randbelow(c.sz[r2] + 1);
  c.insert(r2, pos, v);
}

__device__ __forceinline__ void pop_reverse(PartCtx& c) {
  const int r = c.pick_row(2);
  if (r < 0) return;
  const int size = c.sz[r];
  const int i = c.randbelow(size - 1);
  const int j = c.randrange(i + 1, size);
  const int s = c.start(r);
  rev_short(c.cells, s + i, s + j);
}

__device__ __forceinline__ void pop_or_opt(PartCtx& c) {
  const int L = c.randrange(2, 4);
  const int r1 = c.pick_row(L);  // partition: min size L (operators.py:267)
  if (r1 < 0) return;
  const int st = c.randbelow(c.sz[r1] - L + 1);
  int cnt = 0;
  for (int r = 0; r < c.d1; ++r) cnt += r == r1 || c.sz[r] + L <= c.d2;
  int k = c.randbelow(cnt), r2 = r1;
  for (int r = 0; r < c.d1; ++r)
    if ((r == r1 || c.sz[r] + L <= c.d2) && k-- == 0) {
      r2 = r;
      break;
    }
  short seg[3];
  for (int t = 0; t < L; ++t) seg[t] = c.remove(r1, st);
  const int pos = c.randbelow(c.sz[r2] + 1);
  for (int t = 0; t < L; ++t) c.insert(r2, pos + t, seg[t]);
}

__device__ __forceinline__ void pop_three_opt(PartCtx& c) {
  const int r = c.pick_row(4);
  if (r < 0) {
    pop_reverse(c);
    return;
  }
  const int size = c.sz[r];
  int i, j, k;
  sample3_sorted(c, size, i, j, k);  // sample(range(1, size), 3), sorted
  const int variant = c.randbelow(7);
  short* a = c.cells + c.start(r);
  switch (variant) {
    case 0: rev_short(a, i, j - 1); break;
    case 1: rev_short(a, j, k - 1); break;
    case 2: rev_short(a, i, j - 1); rev_short(a, j, k - 1); break;
    case 3:
    case 4:
    case 5: {
      rev_short(a, i, j - 1);
      rev_short(a, j, k - 1);
      rev_short(a, i, k - 1);
      const int lc = k - j;
      if (variant == 4) rev_short(a, i + lc, k - 1);
      if (variant == 5) rev_short(a, i, i + lc - 1);
      break;
    }
    default: rev_short(a, i, k - 1); break;
  }
}

__device__ __forceinline__ void pop_row_swap(PartCtx& c) {
  if (c.d1 < 2) return;
  int r1 = c.randbelow(c.d1);
  int r2 = c.randbelow(c.d1 - 1);
  r2 += r2 >= r1;
  if (r1 > r2) {
    const int t = r1;
    r1 = r2;
    r2 = t;
  }
  const int sa = c.start(r1), la = c.sz[r1], sb = c.start(r2), lb = c.sz[r2];
  const int lm = sb - (sa + la);
  rev_short(c.cells, sa, sb + lb - 1);  // A M B -> B^r M^r A^r
  rev_short(c.cells, sa, sa + lb - 1);
  rev_short(c.cells, sa + lb, sa + lb + lm - 1);
  rev_short(c.cells, sa + lb + lm, sb + lb - 1);
  c.sz[r1] = (short)lb;
  c.sz[r2] = (short)la;
}

__device__ __forceinline__ void pop_row_split(PartCtx& c) {
  const int r = c.pick_row(2);
  if (r < 0) return;
  const int size = c.sz[r];
  const int cut = c.randrange(1, size);
  const int tl = size - cut;
  int ne = 0, nr = 0;
  for (int t = 0; t < c.d1; ++t) {
    if (t == r) continue;
    ne += c.sz[t] == 0;
    nr += c.sz[t] > 0 && c.sz[t] + tl <= c.d2;
  }
  const bool use_empty = ne > 0;
  const int cnt = use_empty ? ne : nr;
  if (cnt == 0) return;
  int k = c.randbelow(cnt), t = -1;
  for (int q = 0; q < c.d1; ++q) {
    if (q == r) continue;
    const bool ok = use_empty ? c.sz[q] == 0 : (c.sz[q] > 0 && c.sz[q] + tl <= c.d2);
    if (ok && k-- == 0) {
      t = q;
      break;
    }
  }
  // move the tail block to the end of row t
  const int a = c.start(r) + cut;
  const int end_t = c.start(t) + c.sz[t];  // insertion point in the full array
  const int b = end_t > a ? end_t - tl : end_t;
  move_block(c.cells, a, tl, b);
  c.sz[r] = (short)cut;
  c.sz[t] = (short)(c.sz[t] + tl);
}

__device__ __forceinline__ void pop_row_merge(PartCtx& c) {
  int order[64];
  int m = 0;
  for (int r = 0; r < c.d1 && m < 64; ++r)
    if (c.sz[r] > 0) order[m++] = r;
  if (m < 2) return;
  for (int i = m - 1; i >= 1; --i) {  // random.shuffle
    const int j = c.randbelow(i + 1);
    const int t = order[i];
    order[i] = order[j];
    order[j] = t;
  }
  for (int x = 0; x < m; ++x)
    for (int y = 0; y < m; ++y) {
      const int a = order[x], b = order[y];
      if (a != b && c.sz[a] + c.sz[b] <= c.d2) {
        const int sb = c.start(b), lb = c.sz[b];
        const int end_a = c.start(a) + c.sz[a];
        const int dst = end_a > sb ? end_a - lb : end_a;
        move_block(c.cells, sb, lb, dst);
        c.sz[a] = (short)(c.sz[a] + lb);
        c.sz[b] = 0;
        return;
      }
    }
}

__device__ __forceinline__ void pop_seg_shuffle(PartCtx& c) {
  const int r = c.pick_row(2);
  if (r < 0) return;
  const int size = c.sz[r];
  const int ls = lns_scope(c.n_cfg);
  const int len = ls < size ? ls : size;
  const int s0 = c.randbelow(size - len + 1);
  short* seg = c.cells + c.start(r) + s0;
  for (int i = len - 1; i >= 1; --i) {
    const int j = c.randbelow(i + 1);
    const short t = seg[i];
    seg[i] = seg[j];
    seg[j] = t;
  }
}

__device__ __forceinline__ void pop_scatter_shuffle(PartCtx& c) {
  // global cells == compact indices, so the single-row port applies verbatim
  RowCtx<short> rc;
  rc.rng = c.rng;
  rc.row = c.cells;
  rc.n = c.total;
  rc.n_cfg = c.n_cfg;
  short dummy[MAX_RANGES * 2];
  rc.rlo = dummy;
  rc.rhi = dummy + MAX_RANGES;
  rc.rstride = 1;
  rc.nr = 0;
  rc.err = 0;
  rc.full = c.cells;
  rc.d1 = 1;
  rc.d2 = c.total;
  rc.mf = 0;
  rop_scatter_shuffle(rc);
  c.rng = rc.rng;
}

// op_ox_crossover, MULTI_PARTITION branch (operators.py:437-448): OX over the
// flattened active values, written back with the row sizes unchanged.  The
// compact cells ARE the flattened values, and every mate holds all n cells.
__device__ __forceinline__ void pop_ox(PartCtx& c) {
  const short* mate = c.mates->pick(c);
  if (mate == nullptr) return;
  if (c.total < 2) return;
  ox_in_place(c.cells, mate, c.total, c);
}

__device__ __forceinline__ void run_part_op(int kind, PartCtx& c) {
  switch (kind) {
    case SEQ_SWAP: pop_swap(c); break;
    case SEQ_INSERT: pop_insert(c); break;
    case SEQ_REVERSE: pop_reverse(c); break;
    case SEQ_OR_OPT: pop_or_opt(c); break;
    case SEQ_THREE_OPT: pop_three_opt(c); break;
    case SEQ_ROW_SWAP: pop_row_swap(c); break;
    case SEQ_ROW_SPLIT: pop_row_split(c); break;
    case SEQ_ROW_MERGE: pop_row_merge(c); break;
    case SEQ_SEG_SHUFFLE: pop_seg_shuffle(c); break;
    case SEQ_SCATTER_SHUFFLE: pop_scatter_shuffle(c); break;
    case SEQ_OX: pop_ox(c); break;
    default: c.err |= ERR_UNKNOWN_SEQ;
  }
}

// ---- exact evaluation --------------------------------------------------------------
// numpy pairwise_sum (loops_utils.h) over f(lo .. lo+n-1); matches np.sum bit-for-bit.
// Blocks of <= 128 elements are summed inline (the functor stays in registers);
// only longer ranges take the recursive split, out of line.
template <class F>
__device__ __forceinline__ double np_pairwise_leaf(const F& f, int lo, int n) {
  if (n < 8) {
    double res = -0.0;
#pragma unroll 1
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, f(lo + i));
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = f(lo + j);
  int i = 8;
#pragma unroll 1
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f(lo + i + j));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
#pragma unroll 1
  for (; i < n; ++i) res = __dadd_rn(res, f(lo + i));
  return res;
}
template <class F>
__device__ double np_pairwise_split(const F& f, int lo, int n);
template <class F>
__device__ __forceinline__ double np_pairwise(const F& f, int lo, int n) {
  return n <= 128 ? np_pairwise_leaf(f, lo, n) : np_pairwise_split(f, lo, n);
}
template <class F>
__device__ double np_pairwise_split(const F& f, int lo, int n) {
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(np_pairwise(f, lo, n2), np_pairwise(f, lo + n2, n - n2));
}

// CPython 3.12 builtin sum over floats (Neumaier, start 0): streaming form
struct PySum {
  double s, c;
  int first;
  __device__ __forceinline__ void init() {
    s = 0.0;
    c = 0.0;
    first = 1;
  }
  __device__ __forceinline__ void add(double x) {
    if (first) {
      s = x;
      first = 0;
      return;
    }
    const double t = __dadd_rn(s, x);
    if (fabs(s) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(s, t), x));
    else c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), s));
    s = t;
  }
  __device__ __forceinline__ double result() const {
    if (first) return 0.0;
    return (c != 0.0 && isfinite(c)) ? __dadd_rn(s, c) : s;
  }
};

// a route of a compact partition row with one value virtually inserted
struct RouteIns {
  const short* base;
  int ins, v;  // ins < 0: no insertion
  __device__ __forceinline__ int operator[](int q) const {
    return ins < 0 || q < ins ? base[q] : (q == ins ? v : base[q - 1]);
  }
};
struct EdgeV {
  const double* d;
  RouteIns r;
  int n1;
  __device__ __forceinline__ double operator()(int i) const {
    return d[(r[i] + 1) * n1 + r[i + 1] + 1];
  }
};
struct DemV {
  const double* dem;
  RouteIns r;
  __device__ __forceinline__ double operator()(int i) const { return dem[r[i]]; }
};

// part_eval (go_part.cuh) of the row with v inserted at (ri, pi): the same
// arithmetic in the same order, element access through RouteIns.  Out of line:
// one copy for the lane evaluation, the guided-rebuild trials and the cache build
// (the inlined copies were a third of the partition kernel's instructions).
struct PartEval {
  double distance, penalty;
  int veh;
};
__device__ __noinline__ PartEval part_eval_ins(const PartView& v, const short* cells,
                                               const short* sz, int ri, int pi, int val) {
  const int n1 = v.n + 1;
  int veh = 0;
  for (int r = 0; r < v.d1; ++r) veh += (sz[r] + (r == ri)) > 0;
  PySum dsum;
  dsum.init();
  double cap_pen = 0.0, late = 0.0;
  int at = 0;
  double nl_total = 0.0;  // vrp_nonlinear: one running sum over every edge
  long long viol = 0;     // vrp_priority: precedence violations
  for (int r = 0; r < v.d1; ++r) {
    const int len0 = sz[r];
    RouteIns route{cells + at, r == ri ? pi : -1, val};
    const int len = len0 + (r == ri);
    if (v.variant == 2) {  // NonlinearVrpProblem.compute_objective (builtins.py:219-237)
      if (len > 0) {
        double load = 0.0;
        int prev = 0;
        for (int q = 0; q < len; ++q) {
          const int c = route[q], node = c + 1;
          const double x = __ddiv_rn(load, v.cap);
          const double f = __dadd_rn(1.0, __dmul_rn(0.3, __dmul_rn(x, x)));
          nl_total = __dadd_rn(nl_total, __dmul_rn(v.dist[prev * n1 + node], f));
          load = __dadd_rn(load, v.demand[c]);
          prev = node;
        }
        const double x = __ddiv_rn(load, v.cap);
        const double f = __dadd_rn(1.0, __dmul_rn(0.3, __dmul_rn(x, x)));
        nl_total = __dadd_rn(nl_total, __dmul_rn(v.dist[prev * n1], f));
      }
    } else {
      double rd = 0.0;
      if (len > 0) {
        rd = __dadd_rn(v.dist[route[0] + 1], v.dist[(route[len - 1] + 1) * n1]);
        if (len > 1) {
          EdgeV e{v.dist, route, n1};
          rd = __dadd_rn(rd, np_pairwise(e, 0, len - 1));
        }
      }
      dsum.add(rd);
    }
    if (v.variant == 1)  // PriorityVrpProblem.compute_penalty (builtins.py:203-210)
      for (int a = 0; a < len; ++a) {
        const double pa = v.prio[route[a]];
        for (int b = a + 1; b < len; ++b) viol += v.prio[route[b]] > pa;
      }
    DemV dm{v.demand, route};
    const double load = np_pairwise(dm, 0, len);
    const double over = __dsub_rn(load, v.cap);
    cap_pen = __dadd_rn(cap_pen, over > 0.0 ? over : 0.0);
    if (v.tw && len > 0) {
      double t = v.ready[0];
      int prev = 0;
      for (int q = 0; q < len; ++q) {
        const int node = route[q] + 1;
        const double arr0 = __dadd_rn(t, v.dist[prev * n1 + node]);
        const double arrival = v.ready[node] >= arr0 ? v.ready[node] : arr0;
        const double lt = __dsub_rn(arrival, v.due[node]);
        late = __dadd_rn(late, lt > 0.0 ? lt : 0.0);
        t = __dadd_rn(arrival, v.service[node]);
        prev = node;
      }
      const double back = __dsub_rn(__dadd_rn(t, v.dist[prev * n1]), v.due[0]);
      late = __dadd_rn(late, back > 0.0 ? back : 0.0);
    }
    at += len0;
  }
  PartEval e;
  e.distance = v.variant == 2 ? nl_total : dsum.result();
  e.penalty = v.tw ? __dadd_rn(cap_pen, late) : cap_pen;
  if (v.variant == 1) e.penalty = __dadd_rn(e.penalty, (double)viol);
  e.veh = veh;
  return e;
}

// Φ parts of a compact partition row: distance objective and penalty
// (+ the "vehicles" objective, builtins.py:133: non-empty routes)
__device__ __forceinline__ void part_eval(const PartView& v, const short* cells, const short* sz,
                                          double& distance, double& penalty, int* veh = nullptr) {
  const PartEval e = part_eval_ins(v, cells, sz, -1, 0, 0);
  distance = e.distance;
  penalty = e.penalty;
  if (veh) *veh = e.veh;
}

}  // namespace go
