// go_row.cuh — single-row operators on a lane-private materialised row.
//
// Used by the row kernel (go_evolve_row.cuh) for QAP (permutation), knapsack
// (binary) and JSP-int (integer).  Each operator is a direct port of the
// reference (operators.py line cited) acting on the lane's own copy of the
// row, drawing from the lane stream in the reference's order (including
// _pick_row's randrange(1) and CPython's sample()/shuffle() algorithms), and
// records the position ranges it touched so evaluation can be incremental.
#pragma once
#include "go_common.cuh"

namespace go {

enum { MAX_RANGES = 6 };

template <class G>
struct RowCtx {
  Stream rng;  // by value: a pointer would pin the stream to (L2-backed) local memory
  G* row;
  int n;         // active length (== d2 for single-row problems)
  int n_cfg;     // ProblemConfig.n (lns_scope argument)
  int lb, ub;    // integer encoding bounds
  int nr;        // ranges recorded, > MAX_RANGES means "whole row"
  short* rlo;    // lane-state range arrays in shared memory (stride `rstride`)
  short* rhi;
  int rstride;
  int err;
  const MateSel* mates;  // crossover mates (engine.py:553-559)
  // MULTI_FIXED rows (user problems): `full` holds d1 rows of d2 genes; mf = 1
  // permutation rows (ops act on one row, n = d2), mf = 2 binary / integer cells
  // (cell ops act on all d1*d2 cells, segment ops on one row)
  G* full;
  int d1, d2, mf;

  // _pick_row (operators.py:140-144): every row holds d2 genes, so the draw is
  // randrange(d1) (randrange(1) for single-row problems); the op continues on
  // that row
  __device__ __forceinline__ int pick_row() {
    const int r = rng.randbelow(d1);
    if (mf) {
      row = full + r * d2;
      n = d2;
    }
    return r;
  }
  __device__ __forceinline__ int row_len() const { return mf ? d2 : n; }

  __device__ __forceinline__ void mark(int lo, int hi) {
    if (nr < MAX_RANGES) {
      rlo[nr * rstride] = (short)lo;
      rhi[nr * rstride] = (short)hi;
    }
    ++nr;
  }
  __device__ __forceinline__ void mark_all() { nr = MAX_RANGES + 1; }
  __device__ __forceinline__ int randbelow(int m) { return rng.randbelow(m); }
  __device__ __forceinline__ int randrange(int lo, int hi) { return rng.randrange(lo, hi); }
};

template <class G>
__device__ __forceinline__ void row_reverse_range(G* r, int i, int j) {  // [i, j]
  while (i < j) {
    const G t = r[i];
    r[i] = r[j];
    r[j] = t;
    ++i;
    --j;
  }
}

// remove at i, reinsert at j of the shortened row (len n)
template <class G>
__device__ __forceinline__ void row_move_one(G* r, int i, int j) {
  const G v = r[i];
  if (j > i) {
    for (int p = i; p < j; ++p) r[p] = r[p + 1];
  } else {
    for (int p = i; p > j; --p) r[p] = r[p - 1];
  }
  r[j] = v;
}

// ---- permutation ops (operators.py:205-315) -----------------------------------
template <class G>
__device__ __forceinline__ void rop_swap(RowCtx<G>& c) {
  const int n = c.n;
  if (n < 2) return;
  c.pick_row();
  const int i = c.randbelow(n);
  int j = c.randbelow(n - 1);
  j += j >= i;
  const G t = c.row[i];
  c.row[i] = c.row[j];
  c.row[j] = t;
  c.mark(i, i + 1);
  c.mark(j, j + 1);
}

template <class G>
__device__ __forceinline__ void rop_insert(RowCtx<G>& c) {
  const int n = c.n;
  if (n < 2) return;
  c.pick_row();
  const int i = c.randbelow(n);
  const int j = c.randbelow(n);
  row_move_one(c.row, i, j);
  c.mark(i < j ? i : j, (i < j ? j : i) + 1);
}

template <class G>
__device__ __forceinline__ void rop_reverse(RowCtx<G>& c) {
  const int n = c.n;
  if (n < 2) return;
  c.pick_row();
  const int i = c.randbelow(n - 1);
  const int j = c.randrange(i + 1, n);
  row_reverse_range(c.row, i, j);
  c.mark(i, j + 1);
}

template <class G>
__device__ __forceinline__ void rop_or_opt(RowCtx<G>& c) {
  const int L = c.randrange(2, 4);
  const int n = c.n;
  if (n < L + 1) return;
  c.pick_row();
  const int s = c.randbelow(n - L + 1);
  G seg[3];
  for (int t = 0; t < L; ++t) seg[t] = c.row[s + t];
  for (int p = s; p < n - L; ++p) c.row[p] = c.row[p + L];  // remove
  const int pos = c.randbelow(n - L + 1);
  for (int p = n - 1; p >= pos + L; --p) c.row[p] = c.row[p - L];  // open the gap
  for (int t = 0; t < L; ++t) c.row[pos + t] = seg[t];
  c.mark(s < pos ? s : pos, (s < pos ? pos : s) + L);
}

template <class G>
__device__ __forceinline__ void rop_three_opt(RowCtx<G>& c) {
  const int n = c.n;
  if (n < 4) {  // _pick_row(sol, rng, 4) is None -> op_reverse (operators.py:292-294)
    rop_reverse(c);
    return;
  }
  c.pick_row();
  int i, j, k;
  sample3_sorted(c, n, i, j, k);
  const int variant = c.randbelow(7);
  G* r = c.row;
  // a=[0,i) b=[i,j) c=[j,k) d=[k,n): reversals / rotations in place
  switch (variant) {
    case 0: row_reverse_range(r, i, j - 1); break;                         // a b^r c d
    case 1: row_reverse_range(r, j, k - 1); break;                         // a b c^r d
    case 2: row_reverse_range(r, i, j - 1); row_reverse_range(r, j, k - 1); break;
    case 3:                                                                // a c b d
    case 4:                                                                // a c b^r d
    case 5: {                                                              // a c^r b d
      row_reverse_range(r, i, j - 1);
      row_reverse_range(r, j, k - 1);
      row_reverse_range(r, i, k - 1);  // rotation: c b
      const int lc = k - j;
      if (variant == 4) row_reverse_range(r, i + lc, k - 1);
      if (variant == 5) row_reverse_range(r, i, i + lc - 1);
      break;
    }
    default: row_reverse_range(r, i, k - 1); break;                       // a c^r b^r d
  }
  c.mark(i, k);
}

// ---- binary / integer ops (operators.py:318-354) --------------------------------
template <class G>
__device__ __forceinline__ void rop_flip(RowCtx<G>& c) {
  if (c.n == 0) return;
  const int p = c.randbelow(c.n);  // _pick_cell
  c.row[p] = (G)(1 - c.row[p]);
  c.mark(p, p + 1);
}

template <class G>
__device__ __forceinline__ void rop_seg_flip(RowCtx<G>& c) {
  if (c.row_len() < 1) return;
  c.pick_row();
  const int n = c.n;
  const int i = c.randbelow(n);
  const int j = c.randrange(i, n);
  for (int p = i; p <= j; ++p) c.row[p] = (G)(1 - c.row[p]);
  c.mark(i, j + 1);
}

template <class G>
__device__ __forceinline__ void rop_random_reset(RowCtx<G>& c) {
  if (c.n == 0) return;
  const int p = c.randbelow(c.n);
  c.row[p] = (G)c.randrange(c.lb, c.ub + 1);
  c.mark(p, p + 1);
}

template <class G>
__device__ __forceinline__ void rop_seg_reset(RowCtx<G>& c) {
  if (c.row_len() < 1) return;
  c.pick_row();
  const int n = c.n;
  const int i = c.randbelow(n);
  const int j = c.randrange(i, n);
  for (int p = i; p <= j; ++p) c.row[p] = (G)c.randrange(c.lb, c.ub + 1);
  c.mark(i, j + 1);
}

// ---- crossover (operators.py:412-462) -------------------------------------------
// _ox_sequence in place: the kept slice [c1, c2] stays, the other positions are
// refilled in cyclic order from c2+1 with the mate's values (rotated to start
// after c2) that are not in the slice.  Mate rows are read from the snapshot
// with ld.global.cg (written by other SMs during this launch).
// Membership of values < 128 in four registers (selects, no local memory).
struct Bits128 {
  u32 b0, b1, b2, b3;
  __device__ __forceinline__ void clear() { b0 = b1 = b2 = b3 = 0u; }
  __device__ __forceinline__ void set(int v) {
    const u32 w = (u32)v >> 5, m = 1u << (v & 31);
    b0 |= w == 0 ? m : 0u;
    b1 |= w == 1 ? m : 0u;
    b2 |= w == 2 ? m : 0u;
    b3 |= w == 3 ? m : 0u;
  }
  __device__ __forceinline__ bool test(int v) const {
    const u32 w = (u32)v >> 5;
    const u32 x = w == 0 ? b0 : (w == 1 ? b1 : (w == 2 ? b2 : (w == 3 ? b3 : 0u)));
    return (x >> (v & 31)) & 1u;
  }
};

template <class G, class R>
__device__ __forceinline__ void ox_in_place(G* row, const short* mate, int n, R& rng) {
  int c1 = rng.randbelow(n), c2 = rng.randbelow(n);
  if (c1 > c2) {
    const int t = c1;
    c1 = c2;
    c2 = t;
  }
  int w = c2 + 1 == n ? 0 : c2 + 1;  // next free position
  int src = w;
  Bits128 kept;
  kept.clear();
  bool small = n <= 128;  // slice membership as a bit set: O(n) instead of O(n * slice)
  if (small) {
#pragma unroll 1
    for (int q = c1; q <= c2; ++q) {
      const int v = (int)row[q];
      small &= (unsigned)v < 128u;
      kept.set(v);
    }
  }
  for (int t0 = 0; t0 < n; t0 += 8) {  // 8 mate loads in flight per batch
    G mv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (t0 + i < n) mv[i] = (G)__ldcg(mate + src);
      src = src + 1 == n ? 0 : src + 1;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (t0 + i >= n) break;
      const G v = mv[i];
      bool in_slice = false;
      if (small) {
        in_slice = kept.test((int)v);
      } else {
#pragma unroll 1
        for (int q = c1; q <= c2; ++q) in_slice |= row[q] == v;
      }
      if (in_slice) continue;
      row[w] = v;
      w = w + 1 == n ? 0 : w + 1;
      if (w == c1) w = c2 + 1 == n ? 0 : c2 + 1;  // never lands inside the slice
    }
  }
}

template <class G>
__device__ __forceinline__ void rop_ox(RowCtx<G>& c) {
  const short* mate = c.mates->pick(c);
  if (mate == nullptr) return;
  // SINGLE_SEQ: row 0 without a draw; MULTI_FIXED: randrange(d1) (operators.py:450)
  const int off = c.mf == 1 ? c.pick_row() * c.d2 : 0;
  if (c.n < 2) return;
  ox_in_place(c.row, mate + off, c.n, c);
  c.mark_all();
}

template <class G>
__device__ __forceinline__ void rop_uniform_x(RowCtx<G>& c) {
  const short* mate = c.mates->pick(c);
  if (mate == nullptr) return;
  int lo = c.n, hi = 0;
  for (int p0 = 0; p0 < c.n; p0 += 8) {  // draws first, then 8 mate loads in flight
    unsigned take = 0;
    for (int i = 0; i < 8 && p0 + i < c.n; ++i) take |= (c.rng.random() < 0.5 ? 1u : 0u) << i;
    G mv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (take >> i & 1u) mv[i] = (G)__ldcg(mate + p0 + i);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (take >> i & 1u) {
        c.row[p0 + i] = mv[i];
        lo = p0 + i < lo ? p0 + i : lo;
        hi = p0 + i + 1;
      }
  }
  if (hi > lo) c.mark(lo, hi);
}

// ---- LNS shuffles (operators.py:468-499) -----------------------------------------
template <class G>
__device__ __forceinline__ void rop_seg_shuffle(RowCtx<G>& c) {
  if (c.row_len() < 2) return;
  c.pick_row();
  const int n = c.n;
  const int len = lns_scope(c.n_cfg) < n ? lns_scope(c.n_cfg) : n;
  const int s = c.randbelow(n - len + 1);
  G* seg = c.row + s;
  for (int i = len - 1; i >= 1; --i) {  // random.shuffle
    const int j = c.randbelow(i + 1);
    const G t = seg[i];
    seg[i] = seg[j];
    seg[j] = t;
  }
  c.mark(s, s + len);
}

template <class G>
__device__ __forceinline__ void rop_scatter_shuffle(RowCtx<G>& c) {
  if (c.mf == 1) c.pick_row();  // permutation rows: one row (operators.py:481-494)
  const int total = c.n;
  if (total < 2) return;
  int m = lns_scope(c.n_cfg);
  if (m > total) m = total;
  int picks[30];
  G vals[30];
  sample_range(c, total, m, picks);  // random.sample(range(total), m)
  for (int t = 0; t < m; ++t) vals[t] = c.row[picks[t]];
  for (int i = m - 1; i >= 1; --i) {
    const int j = c.randbelow(i + 1);
    const G t = vals[i];
    vals[i] = vals[j];
    vals[j] = t;
  }
  for (int t = 0; t < m; ++t) c.row[picks[t]] = vals[t];
  c.mark_all();
}

template <class G>
__device__ __forceinline__ void run_row_op(int kind, RowCtx<G>& c) {
  switch (kind) {
    case SEQ_SWAP: rop_swap(c); break;
    case SEQ_INSERT: rop_insert(c); break;
    case SEQ_REVERSE: rop_reverse(c); break;
    case SEQ_OR_OPT: rop_or_opt(c); break;
    case SEQ_THREE_OPT: rop_three_opt(c); break;
    case SEQ_FLIP: rop_flip(c); break;
    case SEQ_SEG_FLIP: rop_seg_flip(c); break;
    case SEQ_RANDOM_RESET: rop_random_reset(c); break;
    case SEQ_SEG_RESET: rop_seg_reset(c); break;
    case SEQ_SEG_SHUFFLE: rop_seg_shuffle(c); break;
    case SEQ_SCATTER_SHUFFLE: rop_scatter_shuffle(c); break;
    case SEQ_OX: rop_ox(c); break;
    case SEQ_UNIFORM_X: rop_uniform_x(c); break;
    default: c.err |= ERR_UNKNOWN_SEQ;
  }
}

}  // namespace go
