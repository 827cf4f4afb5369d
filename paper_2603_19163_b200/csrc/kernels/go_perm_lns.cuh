// go_perm_lns.cuh — whole-row operators of the permutation (TSP) kernel.
//
// OX crossover, seg/scatter shuffle and guided rebuild (operators.py:412-571)
// rewrite the tour globally, so they cannot be position maps on the shared
// current tour.  A lane that draws one is DEFERRED: after the chain step, one
// warp per deferred lane
//   1. runs the operator — lane 0 of the warp replays the lane's stream from
//      the operator's first draw (the reference's draw order), the warp does
//      the bulk work in its own shared-memory scratch row (OX slice bit set
//      and fill by ballot/prefix, row rotations, first-minimum insertion
//      scans);
//   2. writes the new row once into one of the lane's two global rows (the
//      other may be the chain's own base) and measures it exactly
//      (warp-reduced tour length);
//   3. the lane's chain restarts on it: nm = 0, delta = Φ(row) − Φ(cur).
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

// exact tour length of a materialised row (whole warp; one out-of-line copy)
template <class Policy>
__device__ __noinline__ typename Policy::Acc perm_row_length(const Policy pol, const i16* row,
                                                             int n, int wl) {
  typedef typename Policy::Acc Acc;
  Acc s = 0;
#pragma unroll 1
  for (int p = wl; p < n; p += 32) s += pol.cost_acc(row[p], row[p + 1 == n ? 0 : p + 1]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  return s;
}

// random.sample(range(total), m) on a lane stream, one out-of-line copy for
// the scatter shuffle and guided rebuild (code size: both inline it otherwise)
__device__ __noinline__ Stream sample_range_stream(Stream rng, int total, int m, int* picks,
                                                   int* ovi, int* ovv) {
  sample_range_buf(rng, total, m, picks, ovi, ovv);
  return rng;
}

template <class Acc>
struct DeferRes {
  int changed;
  Acc len;     // exact tour length of the new row (valid when changed)
  Stream rng;  // lane 0: the stream after the operator's draws
};

// One warp resolves one deferred lane.  `dst` is the lane's global row that
// receives the candidate, `wrow` / `wint` the warp's shared-memory scratch
// (a row of n int16 and 32 ints), `C` the lane's chain.  All bulk work runs
// in shared memory and dst is written exactly once:
//   OX        no materialised parent: the kept slice's values are marked in a
//             bit set (wrow), the child is written in one pass over the mate
//             and, on integer matrices, its tour length summed on the way
//   shuffles  parent materialised in wrow, lane 0 permutes it in place
//   rebuild   parked row gathered into wrow straight from the chain, then
//             every re-insertion is a scan + a span rotation in wrow
// `rng` is valid in lane 0 only.  (A register-resident variant of OX / guided
// rebuild was measured 2x slower end to end on C2 in round 1: its unrolled
// shuffle code evicted the evolve loop from the instruction cache.)
template <class Policy>
__device__ __noinline__ DeferRes<typename Policy::Acc> perm_defer(
    const Policy pol, const Chain C, int kind, i16* dst, i16* wrow, int* wint, Stream rng_in,
    const MateSel ms_in, int n_cfg, int wl) {
  typedef typename Policy::Acc Acc;
  const int n = C.n;
  const unsigned FULL = 0xffffffffu;
  DeferRes<Acc> out;
  out.changed = 0;
  out.len = 0;
  // the stream and the mate selector by value (in registers), not through
  // pointers that would pin them to local memory
  Stream& rng_ref = out.rng;
  rng_ref = rng_in;
  Stream* rng = &rng_ref;
  const MateSel ms_v = ms_in;
  const MateSel* ms = &ms_v;
  // ---- draws that precede any row access (lane 0), broadcast to the warp ----
  int a0 = 0, a1 = 0, a2 = 0, live = 0;
  if (wl == 0) {
    if (kind == SEQ_OX) {
      const int mj = ms->pick_index(*rng);
      if (mj >= 0 && n >= 2) {
        a0 = mj;  // mate evolver
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
  live = __shfl_sync(FULL, live, 0);
  if (!live) return out;
  out.changed = 1;

  if (kind == SEQ_OX) {  // _ox_sequence (operators.py:412-425)
#ifdef GO_PHASE_TIMING
    const unsigned long long t_ox0 = clock64();
#endif
    a0 = __shfl_sync(FULL, a0, 0);
    const int c1 = __shfl_sync(FULL, a1, 0), c2 = __shfl_sync(FULL, a2, 0);
    const short* mate = ms->rows + (size_t)a0 * n;
    const int s0 = c2 + 1 == n ? 0 : c2 + 1;
    // rows up to 32 * WINTS values: the slice bit set lives in wint and the mate
    // row, rotated to start at c2+1, is staged into wrow with all its loads in
    // flight at once (one L2 round trip instead of one per 32 values);
    // longer rows keep the bit set in wrow and read the mate from L2
#ifdef GO_NO_OX_STAGE
    const bool staged = false;
#else
    // a shared-memory instance bounds n far below 32 * 32: the staged path is
    // then a compile-time choice and the L2 fallback is not compiled in
    const bool staged = Policy::kInSmem || n <= 32 * 32;
#endif
    unsigned* mask = staged ? (unsigned*)wint : (unsigned*)wrow;
    const int nwords = (n + 31) >> 5;
#pragma unroll 1
    for (int i = wl; i < nwords; i += 32) mask[i] = 0u;
    if (staged) {
#pragma unroll 4
      for (int t = wl; t < n; t += 32) {
        int src = s0 + t;
        src = src >= n ? src - n : src;
        wrow[t] = __ldcg(mate + src);
      }
    }
    __syncwarp();
    // kept slice child[c1..c2] = parent[c1..c2]: copied, marked, inner edges summed
    Acc len = 0;
    int carry = 0, s_first = 0;
    for (int b = c1; b <= c2; b += 32) {
      const int p = b + wl;
      int v = 0;
      if (p <= c2) {
        v = C.at(p);
        dst[p] = (i16)v;
        atomicOr(mask + (v >> 5), 1u << (v & 31));
      }
      if (b == c1) s_first = __shfl_sync(FULL, v, 0);
      int pv = __shfl_up_sync(FULL, v, 1);
      if (wl == 0) pv = carry;
      if (Policy::kIntegral && p <= c2 && p > c1) len += pol.cost_acc(pv, v);
      const int last_lane = c2 - b < 31 ? c2 - b : 31;
      carry = __shfl_sync(FULL, v, last_lane);
    }
    const int s_last = carry;
    __syncwarp();
#ifdef GO_PHASE_TIMING
    const unsigned long long t_ox1 = clock64();
    if (wl == 0) atomicAdd(ms->prof + 30, t_ox1 - t_ox0);  // staging + kept slice
#endif
    // fill: mate values from c2+1 (cyclic) not in the slice, into the free
    // positions from c2+1 (cyclic); with F the fill sequence and S the slice
    // the child read cyclically from c2+1 is F ++ S
    int filled = 0, f_first = -1, f_last = -1;
    const unsigned lt = (1u << wl) - 1u;
#pragma unroll 1
    for (int b = 0; b < n; b += 32) {
      const int t = b + wl;
      int v = 0;
      bool keep = false;
      if (t < n) {
        if (staged) {
          v = wrow[t];
        } else {
          int src = s0 + t;
          src = src >= n ? src - n : src;
          v = __ldcg(mate + src);
        }
        keep = !((mask[v >> 5] >> (v & 31)) & 1u);
      }
      const unsigned bal = __ballot_sync(FULL, keep);
      if (Policy::kIntegral) {
        // previous fill value: the nearest kept lane below, else the last so far
        const unsigned below = bal & lt;
        const int src_lane = below ? 31 - __clz(below) : 0;
        const int pv_in = __shfl_sync(FULL, v, src_lane);
        if (keep && (below || f_last >= 0)) len += pol.cost_acc(below ? pv_in : f_last, v);
        if (bal) {
          const int fv = __shfl_sync(FULL, v, __ffs(bal) - 1);
          const int lv = __shfl_sync(FULL, v, 31 - __clz(bal));
          if (f_first < 0) f_first = fv;
          f_last = lv;
        }
      }
      if (keep) {
        int w = s0 + filled + __popc(bal & lt);
        w = w >= n ? w - n : w;
        dst[w] = (i16)v;
      }
      filled += __popc(bal);
    }
    __syncwarp();
    if (Policy::kIntegral) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) len += __shfl_xor_sync(FULL, len, off);
      if (f_first >= 0) len += pol.cost_acc(f_last, s_first) + pol.cost_acc(s_last, f_first);
      else len += pol.cost_acc(s_last, s_first);
      out.len = len;
    } else {  // float matrices: the materialised row in the usual summation order
      __threadfence_block();
      out.len = perm_row_length(pol, dst, n, wl);
    }
#ifdef GO_PHASE_TIMING
    if (wl == 0) atomicAdd(ms->prof + 31, clock64() - t_ox1);  // fill + length
#endif
    return out;
  }

  const int ls = lns_scope(n_cfg);
  if (kind == SEQ_SEG_SHUFFLE || kind == SEQ_SCATTER_SHUFFLE) {
    // operators.py:468-499; scatter draws its cells before the row is read,
    // then both shuffles permute the parent in place in wrow
    const int m = ls < n ? ls : n;
    if (kind == SEQ_SCATTER_SHUFFLE && wl == 0)
      *rng = sample_range_stream(*rng, n, m, wint, (int*)wrow, (int*)wrow + m);
    __syncwarp();
#pragma unroll 1
    for (int p = wl; p < n; p += 32) wrow[p] = (i16)C.at(p);
    __syncwarp();
    if (wl == 0) {
      if (kind == SEQ_SEG_SHUFFLE) {
        rng->randbelow(1);  // _pick_row(sol, rng, 2) over the single row
        const int s = rng->randbelow(n - m + 1);
        for (int i = m - 1; i >= 1; --i) {
          const int j = rng->randbelow(i + 1);
          const i16 t = wrow[s + i];
          wrow[s + i] = wrow[s + j];
          wrow[s + j] = t;
        }
      } else {  // shuffling values[t] = row[picks[t]] == swapping the picked cells
        for (int i = m - 1; i >= 1; --i) {
          const int j = rng->randbelow(i + 1);
          const int pi = wint[i], pj = wint[j];
          const i16 t = wrow[pi];
          wrow[pi] = wrow[pj];
          wrow[pj] = t;
        }
      }
    }
    __syncwarp();
#pragma unroll 1
    for (int p = wl; p < n; p += 32) dst[p] = wrow[p];
    out.len = perm_row_length(pol, wrow, n, wl);
    return out;
  }

  // ---- guided rebuild (operators.py:501-546), single row, home = None -----------
  // The parked row (survivors in order, then the taken values in pick order)
  // is gathered into wrow straight from the chain; every re-insertion is then
  // one insertion scan of the row without the value (an index skip, two
  // chunks in flight) plus one rotation of the span between its old and new
  // slot.  Lane t tracks the position of taken value t.
  const int m = ls < n - 1 ? ls : n - 1;
  if (wl == 0) *rng = sample_range_stream(*rng, n, m, wint, (int*)wrow, (int*)wrow + m);
  __syncwarp();
  // sorted by (r, -p): descending positions; picks are distinct, so a pick's
  // rank is the number of larger picks
  const int raw = wl < m ? wint[wl] : -1;
  int rank = 0;
  for (int j = 0; j < m; ++j) rank += __shfl_sync(FULL, raw, j) > raw;
  __syncwarp();
  if (wl < m) wint[rank] = raw;
  __syncwarp();
  const int mypick = wl < m ? wint[wl] : 0;
  const int mytaken = wl < m ? C.at(mypick) : 0;
  const int keep = n - m;
  for (int b = 0; b < n; b += 32) {  // gather the parked row into wrow
    const int d = b + wl;
    int src = d;  // d-th survivor: skip picked positions in ascending order
    for (int j = m - 1; j >= 0; --j) src += __shfl_sync(FULL, mypick, j) <= src;
    const int tk = __shfl_sync(FULL, mytaken, d >= keep && d < n ? d - keep : 0);
    if (d < n) wrow[d] = (i16)(d < keep ? C.at(src) : tk);
  }
  __syncwarp();
  i16* aux = wrow;
  int mypos = keep + wl;  // current slot of taken value wl
  const int sz = n - 1;  // trials pos = 0 .. n-1 of the (n-1)-row without v (cyclic tour)
  const int seg = (n + 31) >> 5;  // trial slots per lane
  for (int t = 0; t < m; ++t) {
    const int v = __shfl_sync(FULL, mytaken, t);
    const int q0 = __shfl_sync(FULL, mypos, t);
    auto rv = [&](int i) -> int { return aux[i < q0 ? i : i + 1]; };  // row without v
    // Each lane scans a contiguous run of `seg` slots: the element before a
    // slot is the previous slot's element, already in registers, so the only
    // dependency between slots is the running first-minimum and the loads of
    // a run are all independent (no shuffles in the scan).  Runs are in slot
    // order across lanes, so the (score, slot) reduction below keeps the
    // reference's first minimum.
    typedef typename Policy::Scan Scan;
    Scan best = 0;
    int bp = 0x7fffffff;
    const int s_lo = wl * seg;
    const int s_hi = s_lo + seg < n ? s_lo + seg : n;
    if (s_lo < n) {
      const int first = rv(0);
      // d(prev, v) of slot p is d(v, next) of slot p-1 (symmetric matrices,
      // problems.py:97-107): two matrix reads per slot instead of three
      int pe = rv(s_lo == 0 ? sz - 1 : s_lo - 1);  // element before slot s_lo (cyclic)
      Scan pb = pol.cost_scan(v, pe);
#pragma unroll 2
      for (int p = s_lo; p < s_hi; ++p) {
        const int e = p < sz ? rv(p) : first;
        const Scan b = pol.cost_scan(v, e);
        const Scan c = pol.cost_scan(pe, e);
        // the reference's float64 order: (d(prev,v) + d(v,next)) - d(prev,next)
        const Scan sc = Policy::kIntegral ? pb + b - c
                                          : (Scan)(((double)pb + (double)b) - (double)c);
        if (bp == 0x7fffffff || sc < best) {
          best = sc;
          bp = p;
        }
        pe = e;
        pb = b;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const Scan ob = __shfl_xor_sync(FULL, best, off);
      const int op = __shfl_xor_sync(FULL, bp, off);
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
#pragma unroll 1
  for (int p = wl; p < n; p += 32) dst[p] = aux[p];
  out.len = perm_row_length(pol, aux, n, wl);
  return out;
}

}  // namespace go
