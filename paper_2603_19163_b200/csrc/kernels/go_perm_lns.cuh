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

// row[p .. size-2] = row[p+1 .. size-1]   (whole warp)
__device__ __forceinline__ void warp_pop(i16* row, int size, int p, int wl) {
  for (int b = p; b < size - 1; b += 32) {
    const int q = b + wl;
    const i16 v = q < size - 1 ? row[q + 1] : (i16)0;
    __syncwarp();
    if (q < size - 1) row[q] = v;
    __syncwarp();
  }
}

// row[p+1 .. size] = row[p .. size-1]; row[p] = v   (whole warp)
__device__ __forceinline__ void warp_insert(i16* row, int size, int p, int v, int wl) {
  for (int hi = size; hi > p; hi -= 32) {
    const int q = hi - 1 - wl;
    const i16 x = q >= p ? row[q] : (i16)0;
    __syncwarp();
    if (q >= p) row[q + 1] = x;
    __syncwarp();
  }
  if (wl == 0) row[p] = (i16)v;
  __syncwarp();
}

struct DeferOut {
  int changed;  // 0: the operator was a no-op (no materialisation kept)
};

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
  const int ls = lns_scope(n_cfg);
  const int m = ls < n - 1 ? ls : n - 1;
  int mypick = 0;
  if (wl == 0) {
    int picks[30];
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
    for (int t = 0; t < m; ++t) aux[t] = (i16)picks[t];  // hand the picks to the warp
  }
  __syncwarp();
  if (wl < m) mypick = aux[wl];
  int mytaken = 0, size = n;
  for (int t = 0; t < m; ++t) {  // _row_remove in that order
    const int p = __shfl_sync(0xffffffffu, mypick, t);
    const int v = dst[p];
    if (wl == t) mytaken = v;
    warp_pop(dst, size, p, wl);
    --size;
  }
  if (wl < m) dst[size + wl] = (i16)mytaken;  // park at the row end
  __syncwarp();
  typedef typename Policy::Acc Acc;
  for (int t = 0; t < m; ++t) {
    const int v = __shfl_sync(0xffffffffu, mytaken, t);
    int q0 = 0x7fffffff;  // _locate_value: first occurrence
    for (int b = 0; b < n; b += 32) {
      const unsigned hit = __ballot_sync(0xffffffffu, b + wl < n && dst[b + wl] == v);
      if (hit) {
        q0 = b + __ffs(hit) - 1;
        break;
      }
    }
    warp_pop(dst, n, q0, wl);
    const int sz = n - 1;  // trials pos = 0 .. n-1 of the (n-1)-row (cyclic tour)
    Acc best = 0;
    int bp = 0x7fffffff;
    for (int b = 0; b < n; b += 32) {
      const int pos = b + wl;
      if (pos < n) {
        const int pv = dst[pos == 0 ? sz - 1 : pos - 1];
        const int nx = dst[pos >= sz ? pos - sz : pos];
        const Acc sc = pol.insertion(pv, v, v, nx);
        if (bp == 0x7fffffff || sc < best) {
          best = sc;
          bp = pos;
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
    warp_insert(dst, sz, bp, v, wl);
  }
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
