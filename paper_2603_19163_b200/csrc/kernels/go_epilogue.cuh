// go_epilogue.cuh — one-CTA kernel run between evolve chunks.
//
// It replays, per generation of the chunk, the host-side bookkeeping of the
// reference generation loop (engine.py:703-750) on device state:
//   1. global best: first (generation, evolver) in scan order that is
//      strictly better (core.py:315-347) -> stagnation counter, history,
//      target check (engine.py:703-716);
//   2. AOS barrier every `aos_interval` generations: counters reduced over
//      all evolvers with warp shuffles, EMA + clamp + one normalisation
//      (aos.py:96-134), K-level update (aos.py:137-144), stagnation reset
//      (aos.py:178-186);
//   3. island migration ring / global_top_n / hybrid (engine.py:483-521,
//      :730-743) with the migration stream mix64(seed, 3, event);
//   4. elite injection: worst member <- global best (engine.py:524-532);
//   5. wall-clock deadline from %globaltimer (engine.py:682-684).
// Arithmetic is written in the reference's evaluation order and compiled
// with FMA contraction disabled, so weights are bit-identical to Python's.
#pragma once
#include "go_args.cuh"
#include "go_common.cuh"

namespace go {

enum { EPI_THREADS = 512 };

struct Cand {
  double pen, scal, o0, o1;  // o0/o1: objective vector (multi-objective runs)
  int idx;
};

// comparison keys of a population: penalties, scalarisations and (multi-
// objective runs) objective vectors [P][2]; obj2 == null for single-objective
struct SolKeys {
  const double* pen;
  const double* scal;
  const double* obj2;
  __device__ __forceinline__ Cand at(int i) const {
    Cand x;
    x.pen = pen[i];
    x.scal = scal[i];
    x.o0 = obj2 ? obj2[2 * i] : 0.0;
    x.o1 = obj2 ? obj2[2 * i + 1] : 0.0;
    x.idx = i;
    return x;
  }
};

__device__ __forceinline__ int cand_cmp(const Cand& a, const Cand& b, const MoCmp& mo) {
  return compare_mo(a.pen, a.scal, a.o0, a.o1, b.pen, b.scal, b.o0, b.o1, mo);
}
// a "before" b in best-first order (strictly better, ties -> lower index)
__device__ __forceinline__ bool best_first(const Cand& a, const Cand& b, const MoCmp& mo) {
  const int c = cand_cmp(a, b, mo);
  return c < 0 || (c == 0 && a.idx < b.idx);
}
// a "before" b in worst-first order (strictly worse, ties -> lower index)
__device__ __forceinline__ bool worst_first(const Cand& a, const Cand& b, const MoCmp& mo) {
  const int c = cand_cmp(a, b, mo);
  return c > 0 || (c == 0 && a.idx < b.idx);
}

template <bool WORST>
__device__ Cand block_select(const SolKeys& K, int lo, int hi, const int* excl, int nexcl,
                             Cand* red, const MoCmp& mo) {
  Cand c;
  c.idx = 0x7fffffff;
  c.pen = c.scal = c.o0 = c.o1 = 0;
  if (mo.lex) {
    // Lexicographic comparison with tolerances is not transitive, so the
    // result depends on the scan order: thread 0 scans in index order like
    // best_index / worst_index (engine.py:467-480), strict improvements only
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = lo; i < hi; ++i) {
        bool skip = false;
        for (int e = 0; e < nexcl; ++e) skip |= excl[e] == i;
        if (skip) continue;
        const Cand x = K.at(i);
        if (c.idx == 0x7fffffff || (WORST ? cand_cmp(x, c, mo) > 0 : cand_cmp(x, c, mo) < 0)) c = x;
      }
      red[0] = c;
    }
    __syncthreads();
    const Cand r = red[0];
    __syncthreads();
    return r;
  }
  for (int i = lo + (int)threadIdx.x; i < hi; i += blockDim.x) {
    bool skip = false;
    for (int e = 0; e < nexcl; ++e) skip |= excl[e] == i;
    if (skip) continue;
    const Cand x = K.at(i);
    if (c.idx == 0x7fffffff || (WORST ? worst_first(x, c, mo) : best_first(x, c, mo))) c = x;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    Cand o;
    o.pen = __shfl_xor_sync(0xffffffffu, c.pen, off);
    o.scal = __shfl_xor_sync(0xffffffffu, c.scal, off);
    o.o0 = __shfl_xor_sync(0xffffffffu, c.o0, off);
    o.o1 = __shfl_xor_sync(0xffffffffu, c.o1, off);
    o.idx = __shfl_xor_sync(0xffffffffu, c.idx, off);
    if (o.idx != 0x7fffffff &&
        (c.idx == 0x7fffffff || (WORST ? worst_first(o, c, mo) : best_first(o, c, mo))))
      c = o;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  Cand r = red[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
    const Cand o = red[w];
    if (o.idx != 0x7fffffff &&
        (r.idx == 0x7fffffff || (WORST ? worst_first(o, r, mo) : best_first(o, r, mo))))
      r = o;
  }
  __syncthreads();
  return r;
}

__device__ __forceinline__ void copy_genes(short* dst, const short* src, int W) {
  for (int i = threadIdx.x; i < W; i += blockDim.x) dst[i] = src[i];
}

// ema_weight (aos.py:96-100), evaluated left to right without contraction
__device__ __forceinline__ double ema_w(double w, long long u, long long v, const EpilogueArgs& A) {
  return __dadd_rn(__dmul_rn(A.alpha, w),
                   __dmul_rn(__dsub_rn(1.0, A.alpha),
                             __dadd_rn(__ddiv_rn((double)v, __dadd_rn((double)u, A.eps)), A.floor_)));
}

// CPython 3.12 builtin sum() over floats (Neumaier), start 0
__device__ __forceinline__ double py_sum(const double* x, int n) {
  if (n == 0) return 0.0;
  double s = x[0], c = 0.0;
  for (int i = 1; i < n; ++i) {
    const double t = __dadd_rn(s, x[i]);
    if (fabs(s) >= fabs(x[i])) c = __dadd_rn(c, __dadd_rn(__dsub_rn(s, t), x[i]));
    else c = __dadd_rn(c, __dadd_rn(__dsub_rn(x[i], t), s));
    s = t;
  }
  if (c != 0.0 && isfinite(c)) s = __dadd_rn(s, c);
  return s;
}

__device__ __forceinline__ void island_range(int P, int islands, int i, int& lo, int& hi) {
  const int base = P / islands, extra = P % islands;
  lo = i * base + (i < extra ? i : extra);
  hi = lo + base + (i < extra ? 1 : 0);
}

__device__ __forceinline__ void put_solution_raw(short* genes, double* scal_a, double* pen_a,
                                                 double* obj2, int W, int dst, const short* src,
                                                 const Cand& c) {
  copy_genes(genes + (size_t)dst * W, src, W);
  if (threadIdx.x == 0) {
    pen_a[dst] = c.pen;
    scal_a[dst] = c.scal;
    if (obj2) {
      obj2[2 * dst] = c.o0;
      obj2[2 * dst + 1] = c.o1;
    }
  }
}

__device__ __forceinline__ void put_solution(const EpilogueArgs& A, int dst, const short* src,
                                             const Cand& c) {
  put_solution_raw(A.genes, A.scal, A.pen, A.obj2, A.W, dst, src, c);
}

__device__ __forceinline__ Cand gbest_cand(const GlobalState* gs) {
  Cand c;
  c.pen = gs->gpen;
  c.scal = gs->gscal;
  c.o0 = gs->gobj[0];
  c.o1 = gs->gobj[1];
  c.idx = -1;
  return c;
}

__global__ void __launch_bounds__(EPI_THREADS, 1) go_epilogue_kernel(EpilogueArgs A) {
  __shared__ Cand red[EPI_THREADS / 32];
  __shared__ int s_stop;
  __shared__ Cand s_don[64];
  __shared__ int s_idx[64];
  GlobalState* gs = A.gs;
  if (gs->stop) return;
  const int P = A.P;
  const MoCmp mo = A.mo;
  const SolKeys pop{A.pen, A.scal, A.obj2};

  // ---- 1. per-generation global best / stagnation / target -----------------
  // engine.py:703-708: each evolver in order against the running global best
  // (a population argmin is the same thing unless the comparison is the
  // non-transitive Lexicographic one).  The chunk's per-generation argmins are
  // independent: one warp each, all in flight at once; thread 0 then walks the
  // generations with the global state in registers and writes it back once.
  __shared__ Cand s_gb[MAX_CHUNK];
  __shared__ long long s_last;
  const int ngen = A.ngen < MAX_CHUNK ? A.ngen : MAX_CHUNK;
  if (!mo.lex) {
    const int warp = threadIdx.x >> 5, ln = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int gi = warp; gi < ngen; gi += nw) {
      const SolKeys rec{A.rec_pen + (size_t)gi * P, A.rec_scal + (size_t)gi * P,
                        A.rec_obj2 ? A.rec_obj2 + (size_t)gi * P * 2 : nullptr};
      Cand c;
      c.idx = 0x7fffffff;
      c.pen = c.scal = c.o0 = c.o1 = 0;
      for (int i = ln; i < P; i += 32) {
        const Cand x = rec.at(i);
        if (c.idx == 0x7fffffff || best_first(x, c, mo)) c = x;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        Cand o;
        o.pen = __shfl_xor_sync(0xffffffffu, c.pen, off);
        o.scal = __shfl_xor_sync(0xffffffffu, c.scal, off);
        o.o0 = __shfl_xor_sync(0xffffffffu, c.o0, off);
        o.o1 = __shfl_xor_sync(0xffffffffu, c.o1, off);
        o.idx = __shfl_xor_sync(0xffffffffu, c.idx, off);
        if (o.idx != 0x7fffffff && (c.idx == 0x7fffffff || best_first(o, c, mo))) c = o;
      }
      if (ln == 0) s_gb[gi] = c;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Cand gb = gbest_cand(gs);
    int gev = gs->gev, stop = 0;
    long long ggen = gs->ggen, stall = gs->stall, gens_done = gs->gens_done;
    long long hist_count = gs->hist_count;
    long long last = A.gen0 - 1;
    for (int gi = 0; gi < ngen; ++gi) {
      const long long g = A.gen0 + gi;
      bool improved = false;
      auto take = [&](const Cand& x) {
        gb = x;
        gev = x.idx;
        ggen = g;
        improved = true;
      };
      if (mo.lex) {
        const SolKeys rec{A.rec_pen + (size_t)gi * P, A.rec_scal + (size_t)gi * P,
                          A.rec_obj2 ? A.rec_obj2 + (size_t)gi * P * 2 : nullptr};
        for (int ev = 0; ev < P; ++ev) {
          const Cand x = rec.at(ev);
          if (cand_cmp(x, gb, mo) < 0) take(x);
        }
      } else if (cand_cmp(s_gb[gi], gb, mo) < 0) {
        take(s_gb[gi]);
      }
      if (improved) stall = 0;
      else stall += 1;
      gens_done = g;
      if (A.history && g - 1 < A.hist_cap) {
        A.history[g - 1] = __dadd_rn(gb.scal, __dmul_rn(A.pw, gb.pen));
        hist_count = g;
      }
      last = g;
      if (A.has_target && !(gb.pen > 0.0)) {
        const double v = gb.scal * A.obj_sign_over_w;
        const bool hit = A.obj_sign_over_w > 0 ? v <= A.target + 1e-9 : v >= A.target - 1e-9;
        if (hit) {
          stop = 2;
          break;
        }
      }
    }
    gs->gpen = gb.pen;
    gs->gscal = gb.scal;
    gs->gobj[0] = gb.o0;
    gs->gobj[1] = gb.o1;
    gs->gev = gev;
    gs->ggen = ggen;
    gs->stall = stall;
    gs->gens_done = gens_done;
    gs->hist_count = hist_count;
    s_stop = stop;
    s_last = last;
  }
  __syncthreads();
  const long long last = s_last;
  // the global best's genes: the team best-ever of its evolver.
  // Under the non-transitive Lexicographic comparison a new global best need
  // not be its team's best-ever; those runs use one-generation chunks and take
  // the evolver's current row instead.
  if (gs->gev >= 0) {
    copy_genes(A.gbest_genes, (mo.lex ? A.genes : A.best_genes) + (size_t)gs->gev * A.W, A.W);
    __syncthreads();
    if (threadIdx.x == 0) gs->gev = -1;
  }
  __syncthreads();

  // ---- 2. AOS: aggregate counters, update at the barrier -------------------
  const int nseq = A.reg->nseq;
  {
    const int warp = threadIdx.x >> 5, ln = threadIdx.x & 31, nw = blockDim.x >> 5;
    // values 0..nseq-1 usage, 32.. impr, 64..66 k_usage, 67..69 k_impr
    for (int v = warp; v < 70; v += nw) {
      const int* src;
      int stride, col;
      if (v < 32) { if (v >= nseq) continue; src = A.usage; stride = MAX_SEQ; col = v; }
      else if (v < 64) { if (v - 32 >= nseq) continue; src = A.impr; stride = MAX_SEQ; col = v - 32; }
      else if (v < 67) { src = A.k_usage; stride = 3; col = v - 64; }
      else { src = A.k_impr; stride = 3; col = v - 67; }
      long long s = 0;
      for (int e = ln; e < P; e += 32) s += src[e * stride + col];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (ln == 0) A.agg[v] += s;
    }
  }
  __syncthreads();
  if (!s_stop && last % A.aos_interval == 0 && threadIdx.x == 0) {
    RegistryDev* R = A.reg;
    double pre[32];
    for (int i = 0; i < nseq; ++i) {
      double w = ema_w(R->w[i], A.agg[i], A.agg[32 + i], A);
      double lo = fmax(A.floor_, R->floor_[i]);
      const double hi = fmin(A.cap, R->cap[i]);
      if (hi < lo) lo = hi;
      w = fmin(fmax(w, lo), hi);
      pre[i] = w;
    }
    // weights are np.float64 from here on: plain sequential sums (oracle/aos.py)
    double tot = 0.0;
    for (int i = 0; i < nseq; ++i) tot = __dadd_rn(tot, pre[i]);
    double acc = 0.0;
    for (int i = 0; i < nseq; ++i) {
      R->w[i] = __ddiv_rn(pre[i], tot);
      acc = __dadd_rn(acc, R->w[i]);
      R->cum[i] = acc;
    }
    R->total = acc;
    double nk[3];
    for (int j = 0; j < 3; ++j) nk[j] = fmax(ema_w(R->kw[j], A.agg[64 + j], A.agg[67 + j], A), A.floor_);
    const double kt = py_sum(nk, 3);
    for (int j = 0; j < 3; ++j) R->kw[j] = __ddiv_rn(nk[j], kt);
    if (gs->stall > A.stagnation) {
      R->kw[0] = 0.8;
      R->kw[1] = 0.15;
      R->kw[2] = 0.05;
      gs->stall = 0;
    }
    for (int v = 0; v < 70; ++v) A.agg[v] = 0;
  }
  __syncthreads();

  // ---- 3. island migration ----------------------------------------------------
  if (!s_stop && A.islands >= 2 && last % A.mig_interval == 0) {
    int strat = A.migration;
    if (strat == 2) strat = (gs->mig_events % 2 == 0) ? 0 : 1;
    const int k = A.islands;
    if (strat == 0) {  // ring: donors snapshotted first
      for (int i = 0; i < k; ++i) {
        int lo, hi;
        island_range(P, k, i, lo, hi);
        const Cand b = block_select<false>(pop, lo, hi, nullptr, 0, red, mo);
        copy_genes(A.scratch + (size_t)i * A.W, A.genes + (size_t)b.idx * A.W, A.W);
        if (threadIdx.x == 0) s_don[i] = b;
      }
      __syncthreads();
      for (int i = 0; i < k; ++i) {
        int lo, hi;
        island_range(P, k, (i + 1) % k, lo, hi);
        if (hi - lo == 1) {
          const Cand d = s_don[i];
          if (cand_cmp(d, pop.at(lo), mo) < 0) put_solution(A, lo, A.scratch + (size_t)i * A.W, d);
          __syncthreads();
          continue;
        }
        const Cand w = block_select<true>(pop, lo, hi, nullptr, 0, red, mo);
        const Cand b = block_select<false>(pop, lo, hi, nullptr, 0, red, mo);
        if (w.idx != b.idx) put_solution(A, w.idx, A.scratch + (size_t)i * A.W, s_don[i]);
        __syncthreads();
      }
    } else {  // global_top_n: stable top-n by repeated selection
      const int tn = A.top_n < 64 ? A.top_n : 64;
      int nd = 0;
      for (int d = 0; d < tn && d < P; ++d) {
        const Cand b = block_select<false>(pop, 0, P, s_idx, nd, red, mo);
        copy_genes(A.scratch + (size_t)d * A.W, A.genes + (size_t)b.idx * A.W, A.W);
        if (threadIdx.x == 0) {
          s_idx[d] = b.idx;
          s_don[d] = b;
        }
        __syncthreads();
        nd = d + 1;
      }
      __shared__ int s_slot;
      Stream mr;
      mr.init(mix64_3(A.seed, 3, (u64)gs->mig_events));  // identical in every thread
      for (int i = 0; i < k; ++i) {
        int lo, hi;
        island_range(P, k, i, lo, hi);
        const Cand b = block_select<false>(pop, lo, hi, nullptr, 0, red, mo);
        const int nslots = hi - lo - 1;
        for (int d = 0; d < nd; ++d) {
          if (nslots <= 0) break;
          if (threadIdx.x == 0) {
            int s = lo + mr.randbelow(nslots);
            if (s >= b.idx) ++s;  // slots = members except the island best
            s_slot = s;
          }
          __syncthreads();
          put_solution(A, s_slot, A.scratch + (size_t)d * A.W, s_don[d]);
          __syncthreads();
        }
      }
    }
    if (threadIdx.x == 0) gs->mig_events += 1;
    __syncthreads();
  }

  // ---- 4. elite injection ------------------------------------------------------
  if (!s_stop && last % A.elite_interval == 0) {
    const Cand w = block_select<true>(pop, 0, P, nullptr, 0, red, mo);
    put_solution(A, w.idx, A.gbest_genes, gbest_cand(gs));
  }
  __syncthreads();

  // ---- 5. stop conditions ----------------------------------------------------------
  if (threadIdx.x == 0) {
    int stop = s_stop;
    if (!stop && gs->deadline_ns && (long long)globaltimer() >= gs->deadline_ns) stop = 1;
    if (!stop && last >= A.max_gens) stop = 3;
    if (stop) {
      gs->stop = stop;
      if (A.host_stop) *(volatile int*)A.host_stop = stop;
    }
  }
}

__global__ void go_arm_deadline_kernel(GlobalState* gs, long long budget_ns) {
  gs->deadline_ns = budget_ns > 0 ? (long long)globaltimer() + budget_ns : 0;
}

// snapshot progress of every team := the launch's first generation (EvolveArgs::prog)
__global__ void go_fill_i32_kernel(int* p, int n, int v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

}  // namespace go
