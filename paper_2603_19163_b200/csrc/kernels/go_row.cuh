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
  Stream* rng;
  G* row;
  int n;         // active length (== d2 for single-row problems)
  int n_cfg;     // ProblemConfig.n (lns_scope argument)
  int lb, ub;    // integer encoding bounds
  int nr;        // ranges recorded, > MAX_RANGES means "whole row"
  short* rlo;    // lane-state range arrays in shared memory (stride `rstride`)
  short* rhi;
  int rstride;
  int err;

  __device__ __forceinline__ void mark(int lo, int hi) {
    if (nr < MAX_RANGES) {
      rlo[nr * rstride] = (short)lo;
      rhi[nr * rstride] = (short)hi;
    }
    ++nr;
  }
  __device__ __forceinline__ void mark_all() { nr = MAX_RANGES + 1; }
  __device__ __forceinline__ int randbelow(int m) { return rng->randbelow(m); }
  __device__ __forceinline__ int randrange(int lo, int hi) { return rng->randrange(lo, hi); }
};

// CPython random.sample's table-size rule: set method iff n > setsize
__device__ __forceinline__ int sample_setsize(int k) {
  int s = 21;
  if (k > 5) {
    long long p = 1;
    while (p < 3LL * k) p *= 4;  // 4 ** ceil(log(3k, 4)); 3k is never a power of 4
    s += (int)p;
  }
  return s;
}

// lns_scope (operators.py:130-134): max(2, ceil(min(0.1 n, 30)))
__device__ __forceinline__ int lns_scope(int n) {
  const double x = fmin(0.1 * (double)n, 30.0);
  const int c = (int)ceil(x);
  return c < 2 ? 2 : c;
}

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
  c.randbelow(1);
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
  c.randbelow(1);
  const int i = c.randbelow(n);
  const int j = c.randbelow(n);
  row_move_one(c.row, i, j);
  c.mark(i < j ? i : j, (i < j ? j : i) + 1);
}

template <class G>
__device__ __forceinline__ void rop_reverse(RowCtx<G>& c) {
  const int n = c.n;
  if (n < 2) return;
  c.randbelow(1);
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
  c.randbelow(1);
  const int s = c.randbelow(n - L + 1);
  G seg[3];
  for (int t = 0; t < L; ++t) seg[t] = c.row[s + t];
  for (int p = s; p < n - L; ++p) c.row[p] = c.row[p + L];  // remove
  const int pos = c.randbelow(n - L + 1);
  for (int p = n - 1; p >= pos + L; --p) c.row[p] = c.row[p - L];  // open the gap
  for (int t = 0; t < L; ++t) c.row[pos + t] = seg[t];
  c.mark(s < pos ? s : pos, (s < pos ? pos : s) + L);
}

// sample(range(1, n), 3) sorted (operators.py:300)
template <class G>
__device__ __forceinline__ void sample3_sorted(RowCtx<G>& c, int n, int& i, int& j, int& k) {
  const int N = n - 1;  // population 1..n-1
  int out[3];
  if (N <= sample_setsize(3)) {  // pool method with a virtual pool
    int ovi[3], ovv[3], no = 0;
    for (int t = 0; t < 3; ++t) {
      const int jj = c.randbelow(N - t);
      int val = jj + 1;
      for (int q = 0; q < no; ++q)
        if (ovi[q] == jj) val = ovv[q];
      out[t] = val;
      // pool[jj] = pool[N - t - 1]
      const int src = N - t - 1;
      int sval = src + 1;
      for (int q = 0; q < no; ++q)
        if (ovi[q] == src) sval = ovv[q];
      bool found = false;
      for (int q = 0; q < no; ++q)
        if (ovi[q] == jj) {
          ovv[q] = sval;
          found = true;
        }
      if (!found) {
        ovi[no] = jj;
        ovv[no] = sval;
        ++no;
      }
    }
  } else {  // set method
    for (int t = 0; t < 3; ++t) {
      int jj;
      bool dup;
      do {
        jj = c.randbelow(N);
        dup = false;
        for (int q = 0; q < t; ++q) dup |= (out[q] == jj + 1);
      } while (dup);
      out[t] = jj + 1;
    }
  }
  // sort three
  int a = out[0], b = out[1], d = out[2], t;
  if (a > b) { t = a; a = b; b = t; }
  if (b > d) { t = b; b = d; d = t; }
  if (a > b) { t = a; a = b; b = t; }
  i = a;
  j = b;
  k = d;
}

template <class G>
__device__ __forceinline__ void rop_three_opt(RowCtx<G>& c) {
  const int n = c.n;
  if (n < 4) {  // _pick_row(sol, rng, 4) is None -> op_reverse (operators.py:292-294)
    rop_reverse(c);
    return;
  }
  c.randbelow(1);
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
  const int n = c.n;
  if (n < 1) return;
  c.randbelow(1);
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
  const int n = c.n;
  if (n < 1) return;
  c.randbelow(1);
  const int i = c.randbelow(n);
  const int j = c.randrange(i, n);
  for (int p = i; p <= j; ++p) c.row[p] = (G)c.randrange(c.lb, c.ub + 1);
  c.mark(i, j + 1);
}

// ---- LNS shuffles (operators.py:468-499) -----------------------------------------
template <class G>
__device__ __forceinline__ void rop_seg_shuffle(RowCtx<G>& c) {
  const int n = c.n;
  if (n < 2) return;
  c.randbelow(1);
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
  const int total = c.n;
  if (total < 2) return;
  int m = lns_scope(c.n_cfg);
  if (m > total) m = total;
  int picks[30];
  G vals[30];
  // random.sample(range(total), m)
  if (total <= sample_setsize(m)) {
    int ovi[30], ovv[30], no = 0;
    for (int t = 0; t < m; ++t) {
      const int jj = c.randbelow(total - t);
      int val = jj;
      for (int q = 0; q < no; ++q)
        if (ovi[q] == jj) val = ovv[q];
      picks[t] = val;
      const int src = total - t - 1;
      int sval = src;
      for (int q = 0; q < no; ++q)
        if (ovi[q] == src) sval = ovv[q];
      bool found = false;
      for (int q = 0; q < no; ++q)
        if (ovi[q] == jj) {
          ovv[q] = sval;
          found = true;
        }
      if (!found) {
        ovi[no] = jj;
        ovv[no] = sval;
        ++no;
      }
    }
  } else {
    for (int t = 0; t < m; ++t) {
      int jj;
      bool dup;
      do {
        jj = c.randbelow(total);
        dup = false;
        for (int q = 0; q < t; ++q) dup |= picks[q] == jj;
      } while (dup);
      picks[t] = jj;
    }
  }
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
    default: c.err |= ERR_UNKNOWN_SEQ;
  }
}

}  // namespace go
