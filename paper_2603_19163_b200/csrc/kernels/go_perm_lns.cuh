// go_perm_lns.cuh — whole-row operators of the permutation (TSP) kernel.
//
// OX crossover, seg/scatter shuffle and guided rebuild (operators.py:412-571)
// rewrite the tour globally, so they cannot be position maps on the shared
// current tour.  A lane that draws one is DEFERRED: after the chain step, one
// warp per deferred lane
//   1. materialises the lane's candidate (current tour composed with its
//      chain) into one of the lane's two global rows (the other row may be
//      the chain's own base);
//   2. runs the operator on that row — lane 0 of the warp replays the lane's
//      stream from the operator's first draw (the reference's draw order), the
//      warp does the bulk work (OX fill by ballot/prefix, row shifts, first-
//      minimum insertion scans);
//   3. re-evaluates the row exactly (warp-reduced tour length) and restarts the
//      lane's chain on it: nm = 0, delta = Φ(row) − Φ(cur).
// Guided rebuild scores trials with the insertion delta d(prev,v) + d(v,next)
// − d(prev,next) instead of a full evaluation: on integer matrices Φ(trial) =
// Φ(row without v) + that delta exactly, so first-minimum choices equal the
// reference's full re-evaluations (operators.py:534-545).
#pragma once
#include "go_common.cuh"
#include "go_perm.cuh"

namespace go {

__device__ __forceinline__ bool perm_deferred(int kind) {
  return kind == SEQ_OX || kind == SEQ_SEG_SHUFFLE || kind == SEQ_SCATTER_SHUFFLE ||
         kind == SEQ_GUIDED_REBUILD;
}

// One warp resolves one deferred lane.  `dst` / `aux` are the lane's two
// global rows (dst receives the candidate; aux is scratch), `C` the lane's
// chain (its base may be `aux`).  `rng` is valid in lane 0 only.
template <class Policy>
__device__ __noinline__ int perm_defer_run(const Policy pol, const Chain C, int kind, i16* dst,
                                           i16* aux, Stream* rng, const MateSel* ms, int n_cfg,
                                           int wl) {
  const int n = C.n;
  // ---- draws that precede any row access (lane 0), broadcast to the warp ----
  int a0 = 0, a1 = 0, a2 = 0, live = 0;
  if (wl == 0) {
    if (kind == SEQ_OX) {
      const short* mate = ms->pick(*rng);
      if (mate != nullptr && n >= 2) {
        a0 = (int)((mate - ms->rows) / n);  // mate evolver
        int c1 = rng->randbelow(n), c2 = rng->randbelow(n);
        if (c1 > c2) {
          const int t = c1;
          c1 = c2;
          c2 = t;
        }
        a1 = c1;
        a2 = c2;
        live = 1;
      }
    } else if (kind == SEQ_GUIDED_REBUILD) {
      live = n >= 3;
    } else {
      live = n >= 2;
    }
  }
  live = __shfl_sync(0xffffffffu, live, 0);
  if (!live) return 0;
  a0 = __shfl_sync(0xffffffffu, a0, 0);
  a1 = __shfl_sync(0xffffffffu, a1, 0);
  a2 = __shfl_sync(0xffffffffu, a2, 0);

  // ---- 1. materialise the candidate --------------------------------------------
  for (int p = wl; p < n; p += 32) dst[p] = (i16)C.at(p);
  __syncwarp();

  if (kind == SEQ_OX) {  // _ox_sequence (operators.py:412-425)
    const short* mate = ms->rows + (size_t)a0 * n;
    const int c1 = a1, c2 = a2;
    for (int p = wl; p < n; p += 32) aux[dst[p]] = (i16)p;  // inverse permutation
    __syncwarp();
    const int s0 = c2 + 1 == n ? 0 : c2 + 1;
    int filled = 0;
    for (int b = 0; b < n; b += 32) {
      const int t = b + wl;
      int v = 0;
      bool keep = false;
      if (t < n) {
        int src = s0 + t;
        src = src >= n ? src - n : src;
        v = __ldcg(mate + src);
        const int at = aux[v];
        keep = at < c1 || at > c2;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        int w = s0 + filled + __popc(bal & ((1u << wl) - 1u));
        w = w >= n ? w - n : w;
        dst[w] = (i16)v;
      }
      filled += __popc(bal);
    }
    __syncwarp();
    return 1;
  }
  if (kind == SEQ_SEG_SHUFFLE) {  // operators.py:468-477, lane 0 serial
    if (wl == 0) {
      rng->randbelow(1);  // _pick_row(sol, rng, 2) over the single row
      const int ls = lns_scope(n_cfg);
      const int len = ls < n ? ls : n;
      const int s = rng->randbelow(n - len + 1);
      for (int i = len - 1; i >= 1; --i) {
        const int j = rng->randbelow(i + 1);
        const i16 t = dst[s + i];
        dst[s + i] = dst[s + j];
        dst[s + j] = t;
      }
    }
    __syncwarp();
    return 1;
  }
  if (kind == SEQ_SCATTER_SHUFFLE) {  // operators.py:480-499, lane 0 serial
    if (wl == 0) {
      const int ls = lns_scope(n_cfg);
      const int m = ls < n ? ls : n;
      int picks[30];
      i16 vals[30];
      sample_range(*rng, n, m, picks);
      for (int t = 0; t < m; ++t) vals[t] = dst[picks[t]];
      for (int i = m - 1; i >= 1; --i) {
        const int j = rng->randbelow(i + 1);
        const i16 t = vals[i];
        vals[i] = vals[j];
        vals[j] = t;
      }
      for (int t = 0; t < m; ++t) dst[picks[t]] = vals[t];
    }
    __syncwarp();
    return 1;
  }
  // ---- guided rebuild (operators.py:501-546), single row, home = None -----------
  // One gather builds the parked row (survivors in order, then the taken
  // values in pick order) in `aux`; every re-insertion is then one insertion
  // scan of the row without the value (read through an index skip, two chunks
  // in flight) plus one rotation of the span between its old and new slot.
  // Lane t tracks the position of taken value t, so no search pass is needed.
  const int ls = lns_scope(n_cfg);
  const int m = ls < n - 1 ? ls : n - 1;
  int picks[30];
  if (wl == 0) {
    sample_range(*rng, n, m, picks);
    for (int i = 1; i < m; ++i) {  // sorted by (r, -p): descending positions
      const int v = picks[i];
      int j = i;
      while (j > 0 && picks[j - 1] < v) {
        picks[j] = picks[j - 1];
        --j;
      }
      picks[j] = v;
    }
  }
  int mypick = 0;
  for (int t = 0; t < m; ++t) {
    const int x = __shfl_sync(0xffffffffu, wl == 0 ? picks[t] : 0, 0);
    if (wl == t) mypick = x;
  }
  const int mytaken = wl < m ? dst[mypick] : 0;
  const int keep = n - m;
  for (int b = 0; b < n; b += 32) {  // gather the parked row into aux
    const int d = b + wl;
    int src = d;  // d-th survivor: skip picked positions in ascending order
    for (int j = m - 1; j >= 0; --j) src += __shfl_sync(0xffffffffu, mypick, j) <= src;
    const int pk = __shfl_sync(0xffffffffu, mypick, d >= keep && d < n ? d - keep : 0);
    if (d < n) aux[d] = d < keep ? dst[src] : dst[pk];
  }
  __syncwarp();
  typedef typename Policy::Acc Acc;
  int mypos = keep + wl;  // current slot of taken value wl
  const int sz = n - 1;  // trials pos = 0 .. n-1 of the (n-1)-row without v (cyclic tour)
  for (int t = 0; t < m; ++t) {
    const int v = __shfl_sync(0xffffffffu, mytaken, t);
    const int q0 = __shfl_sync(0xffffffffu, mypos, t);
    auto rv = [&](int i) -> int { return aux[i < q0 ? i : i + 1]; };  // row without v
    const int first = rv(0), last = rv(sz - 1);
    Acc best = 0;
    int bp = 0x7fffffff;
    int carry = last;  // element before slot 0 (cyclic)
    for (int b = 0; b < n; b += 64) {  // two chunks in flight
      const int p0 = b + wl, p1 = b + 32 + wl;
      const int e0 = p0 < sz ? rv(p0) : first;
      const int e1 = p1 < sz ? rv(p1) : first;
      int pv0 = __shfl_up_sync(0xffffffffu, e0, 1);
      int pv1 = __shfl_up_sync(0xffffffffu, e1, 1);
      const int e0_31 = __shfl_sync(0xffffffffu, e0, 31);
      if (wl == 0) {
        pv0 = carry;
        pv1 = e0_31;
      }
      carry = __shfl_sync(0xffffffffu, e1, 31);
      if (p0 < n) {
        const Acc sc = pol.insertion(pv0, v, v, e0);
        if (bp == 0x7fffffff || sc < best) {
          best = sc;
          bp = p0;
        }
      }
      if (p1 < n) {
        const Acc sc = pol.insertion(pv1, v, v, e1);
        if (bp == 0x7fffffff || sc < best) {
          best = sc;
          bp = p1;
        }
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const Acc ob = __shfl_xor_sync(0xffffffffu, best, off);
      const int op = __shfl_xor_sync(0xffffffffu, bp, off);
      if (op != 0x7fffffff && (bp == 0x7fffffff || ob < best || (ob == best && op < bp))) {
        best = ob;
        bp = op;
      }
    }
    // move v from slot q0 to slot bp (the row keeps n slots)
    if (bp < q0) {  // aux[bp+1 .. q0] = aux[bp .. q0-1], high chunks first
      for (int hi = q0; hi > bp; hi -= 64) {
        const int qa = hi - wl, qb = hi - 32 - wl;
        const int xa = qa > bp ? aux[qa - 1] : 0;
        const int xb = qb > bp ? aux[qb - 1] : 0;
        __syncwarp();
        if (qa > bp) aux[qa] = (i16)xa;
        if (qb > bp) aux[qb] = (i16)xb;
        __syncwarp();
      }
      if (mypos >= bp && mypos < q0) ++mypos;
    } else if (bp > q0) {  // aux[q0 .. bp-1] = aux[q0+1 .. bp], low chunks first
      for (int lo = q0; lo < bp; lo += 64) {
        const int qa = lo + wl, qb = lo + 32 + wl;
        const int xa = qa < bp ? aux[qa + 1] : 0;
        const int xb = qb < bp ? aux[qb + 1] : 0;
        __syncwarp();
        if (qa < bp) aux[qa] = (i16)xa;
        if (qb < bp) aux[qb] = (i16)xb;
        __syncwarp();
      }
      if (mypos > q0 && mypos <= bp) --mypos;
    }
    if (wl == 0) aux[bp] = (i16)v;
    if (wl == t) mypos = bp;
    __syncwarp();
  }
  for (int p = wl; p < n; p += 32) dst[p] = aux[p];
  __syncwarp();
  return 1;
}

// exact tour length of a materialised row (whole warp)
template <class Policy>
__device__ __forceinline__ typename Policy::Acc perm_row_length(const Policy& pol, const i16* row,
                                                                int n, int wl) {
  typedef typename Policy::Acc Acc;
  Acc s = 0;
  for (int p = wl; p < n; p += 32) s += pol.cost_acc(row[p], row[p + 1 == n ? 0 : p + 1]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  return s;
}


template <class Acc>
struct DeferRes {
  int changed;
  Acc len;  // exact tour length of the new row (valid when changed)
};

// Runs the deferred operator and measures the new row.  (A register-resident
// variant of OX / guided rebuild was measured 2x slower end to end on C2: its
// unrolled shuffle code evicted the evolve loop from the instruction cache.)
template <class Policy>
__device__ __noinline__ DeferRes<typename Policy::Acc> perm_defer(const Policy pol, const Chain C,
                                                                  int kind, i16* dst, i16* aux,
                                                                  Stream* rng, const MateSel* ms,
                                                                  int n_cfg, int wl) {
  DeferRes<typename Policy::Acc> out;
  out.changed = perm_defer_run(pol, C, kind, dst, aux, rng, ms, n_cfg, wl);
  out.len = out.changed ? perm_row_length(pol, dst, C.n, wl) : 0;
  return out;
}

}  // namespace go
