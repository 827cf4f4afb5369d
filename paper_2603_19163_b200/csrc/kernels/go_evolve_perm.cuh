// go_evolve_perm.cuh — the evolve kernel for single-row permutation problems.
//
// Paper Alg. 1 / reference evolve_generation (engine.py:538-595), B200 layout:
//   * one TEAM of T lanes evolves one solution (the paper's "one block
//     evolves one solution"); E teams share one CTA so that the instance
//     staged once into that CTA's shared memory (cp.async.bulk, up to the
//     227 KB opt-in) serves E evolvers, and each SM keeps 4*E warps resident;
//   * each team synchronises on its own named barrier, never the CTA;
//   * lane work: stream = Philox(mix64(seed, evolver, gen, lane, 0)) ->
//     sample_k -> k x (sample_sequence -> operator -> delta) on the lane's
//     virtual candidate (go_perm.cuh), no per-lane copy;
//   * (delta, lane) argmin with warp shuffles, strict '<' so the lowest lane
//     wins ties (engine.py:578);
//   * SA acceptance with the accept stream (engine.py:584-588);
//   * the winner's move chain is applied by the whole team as a gather
//     new[p] = cur[src(p)] into a ping-pong row;
//   * AOS credit for the winning lane only (engine.py:589-594);
//   * per-generation (pen, scal) records feed the epilogue's global-best /
//     stagnation bookkeeping (engine.py:703-708).
// One launch runs a chunk of generations that never crosses an AOS, elite
// or migration boundary; go_epilogue.cuh runs between chunks.
#pragma once
#include "go_args.cuh"
#include "go_common.cuh"
#include "go_perm.cuh"

namespace go {

struct NoCustomOps {
  template <class Ctx>
  __device__ __forceinline__ static void run(int slot, Ctx& ctx) {
    ctx.err |= ERR_UNKNOWN_SEQ;
  }
};

template <class Acc>
struct TeamShared {
  Acc wd[32];
  int wl[32];
  Move chain[MAX_CHAIN];
  double bd;
  int nm, k, accept, pad;
  int sq[MAX_CHAIN];
  int usage[MAX_SEQ];
  int impr[MAX_SEQ];
  int k_usage[3];
  int k_impr[3];
};

// sample_k (aos.py:147-154)
__device__ __forceinline__ int sample_k(const double* kw, Stream& r) {
  const double x = r.random() * (kw[0] + kw[1] + kw[2]);
  if (x < kw[0]) return 1;
  if (x < kw[0] + kw[1]) return 2;
  return 3;
}

// sample_sequence (aos.py:157-175); cum[] holds the sequential partial sums
__device__ __forceinline__ int sample_seq(const double* cum, int nseq, double total, Stream& r) {
  const double x = r.random() * total;
  for (int i = 0; i < nseq; ++i)
    if (x < cum[i]) return i;
  return nseq - 1;
}

template <class Acc> struct AccMax {
  __device__ __forceinline__ static Acc value() { return (Acc)0x7fffffffffffffffll; }
};
template <> struct AccMax<double> {
  __device__ __forceinline__ static double value() { return 1.7976931348623157e308; }
};

template <class Acc>
__device__ __forceinline__ void argmin_warp(Acc& d, int& l) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const Acc od = __shfl_xor_sync(0xffffffffu, d, off);
    const int ol = __shfl_xor_sync(0xffffffffu, l, off);
    if (od < d || (od == d && ol < l)) {
      d = od;
      l = ol;
    }
  }
}

template <class Policy, class Custom>
__device__ __forceinline__ void run_perm_op(int kind, PermCtx<Policy>& c) {
  switch (kind) {
    case SEQ_SWAP: bi_swap(c); break;
    case SEQ_INSERT: bi_insert(c); break;
    case SEQ_REVERSE: bi_reverse(c); break;
    case SEQ_OR_OPT: bi_or_opt(c); break;
    default:
      if (kind >= SEQ_CUSTOM_BASE) Custom::run(kind - SEQ_CUSTOM_BASE, c);
      else c.err |= ERR_UNKNOWN_SEQ;
  }
}

// Shared-memory carve-up common to the kernel and the host (engine.cu).
struct PermSmem {
  static __host__ __device__ unsigned align(unsigned x, unsigned a) { return (x + a - 1) / a * a; }
  static __host__ __device__ unsigned inst_off() { return 0; }
  static __host__ __device__ unsigned reg_off(unsigned inst_bytes) { return align(inst_bytes, 128); }
  static __host__ __device__ unsigned team_off(unsigned inst_bytes) {
    return reg_off(inst_bytes) + 640;
  }
  static __host__ __device__ unsigned row_bytes(int n) { return align(2u * n, 16); }
  template <class Acc>
  static __host__ __device__ unsigned team_bytes(int n) {
    return align(2 * row_bytes(n) + (unsigned)sizeof(TeamShared<Acc>), 16);
  }
};

template <class Policy, class Custom>
__device__ __forceinline__ void evolve_perm(const EvolveArgs& A, Policy pol) {
  typedef typename Policy::Acc Acc;
  extern __shared__ __align__(128) unsigned char sm[];
  if (A.gs->stop) return;  // uniform: written by an earlier launch

  // ---- stage the instance and the registry --------------------------------
  const unsigned ro = PermSmem::reg_off(A.inst_bytes);
  u64* mbar = (u64*)(sm + ro);
  double* s_cum = (double*)(sm + ro + 16);       // 32 doubles
  double* s_misc = s_cum + 32;                    // kw[3], total
  int* s_kind = (int*)(s_misc + 4);               // 32 ints
  if (A.inst_bytes) {
    stage_to_smem(sm, A.inst, A.inst_bytes, mbar);
    pol.d.m = (const typename decltype(pol.d)::Elem*)sm;
  }
  const RegistryDev* R = A.reg;
  const int nseq = R->nseq;
  for (int i = threadIdx.x; i < 32; i += blockDim.x) {
    s_cum[i] = R->cum[i];
    s_kind[i] = R->kind[i];
  }
  if (threadIdx.x < 3) s_misc[threadIdx.x] = R->kw[threadIdx.x];
  if (threadIdx.x == 3) s_misc[3] = R->total;
  __syncthreads();

  const int TS = A.team_stride, T = A.T, n = A.n;
  const int team = threadIdx.x / TS, lane = threadIdx.x - team * TS;
  const int ev = blockIdx.x * A.E + team;
  if (ev >= A.P) return;  // idle team slot; no CTA-wide barrier follows
  const long long evg = (long long)A.ev_offset + ev;

  unsigned char* tb = sm + PermSmem::team_off(A.inst_bytes) + team * A.team_smem;
  i16* cur = (i16*)tb;
  i16* nxt = (i16*)(tb + PermSmem::row_bytes(n));
  TeamShared<Acc>* ts = (TeamShared<Acc>*)(tb + 2 * PermSmem::row_bytes(n));

  for (int p = lane; p < n; p += TS) cur[p] = A.genes[(size_t)ev * n + p];
  for (int i = lane; i < MAX_SEQ; i += TS) {
    ts->usage[i] = 0;
    ts->impr[i] = 0;
  }
  if (lane < 3) {
    ts->k_usage[lane] = 0;
    ts->k_impr[lane] = 0;
  }
  team_bar(team, TS);

  double phi = A.scal[ev];
  if (A.resync) {  // float matrices: re-anchor Φ on an exact full evaluation
    Acc part = pol.partial(cur, n, lane, TS);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    if ((lane & 31) == 0) ts->wd[lane >> 5] = part;
    team_bar(team, TS);
    Acc tot = 0;
    for (int w = 0; w < TS / 32; ++w) tot += ts->wd[w];
    phi = (double)tot;
    team_bar(team, TS);
  }
  double bscal = A.best_scal[ev], bpen = A.best_pen[ev];
  const double* kw = s_misc;
  const double total = s_misc[3];
  int err = 0;
  unsigned long long rd_pos = 0, rd_elem = 0;

  for (int gi = 0; gi < A.ngen; ++gi) {
    const long long g = A.gen0 + gi;
    const double temp = A.temps[gi];

    // ---- lanes: sample, move, delta --------------------------------------
    Acc delta = 0;
    int k = 0, sq0 = 0, sq1 = 0, sq2 = 0;
    Chain L;
    L.reset(cur, n);
    if (lane < T) {
      Stream rng;
      rng.init(mix64_5(A.seed, (u64)evg, (u64)g, (u64)lane, 0));
      PermCtx<Policy> c;
      c.rng = &rng;
      c.L = &L;
      c.pol = &pol;
      c.err = 0;
      c.rd_pos = 0;
      c.rd_elem = 0;
      k = sample_k(kw, rng);
      for (int s = 0; s < k; ++s) {
        const int si = sample_seq(s_cum, nseq, total, rng);
        if (s == 0) sq0 = si; else if (s == 1) sq1 = si; else sq2 = si;
        c.out.kind = MV_NONE;
        run_perm_op<Policy, Custom>(s_kind[si], c);
        if (c.out.kind != MV_NONE) {
          delta += pol.delta(L, c.out, c.rd_pos, c.rd_elem);
          L.push(c.out);
        }
      }
      err |= c.err;
      rd_pos += c.rd_pos;
      rd_elem += c.rd_elem;
    }

    // ---- team argmin over (delta, lane) ----------------------------------
    Acc bd = lane < T ? delta : AccMax<Acc>::value();  // padding lanes never win
    int bl = lane < T ? lane : 0x7fffffff;
    argmin_warp(bd, bl);
    if ((lane & 31) == 0) {
      ts->wd[lane >> 5] = bd;
      ts->wl[lane >> 5] = bl;
    }
    team_bar(team, TS);
    bd = ts->wd[0];
    bl = ts->wl[0];
    for (int w = 1; w < TS / 32; ++w) {
      const Acc od = ts->wd[w];
      if (od < bd) {  // warps are in lane order: ties keep the lower lane
        bd = od;
        bl = ts->wl[w];
      }
    }
    if (lane == bl) {
      ts->nm = L.nm;
      ts->chain[0] = L.m0;
      ts->chain[1] = L.m1;
      ts->chain[2] = L.m2;
      ts->k = k;
      ts->sq[0] = sq0;
      ts->sq[1] = sq1;
      ts->sq[2] = sq2;
    }
    const double bdd = (double)bd;
    if (lane == 0) {
      int acc = bdd < 0.0;
      if (!acc && temp > 0.0) {
        Stream ar;
        ar.init(mix64_5(A.seed, (u64)evg, (u64)g, 0, 1));
        acc = ar.random() < exp(-bdd / temp);
      }
      ts->accept = acc;
    }
    team_bar(team, TS);

    if (ts->accept) {
      Chain W;
      W.reset(cur, n);
      W.nm = ts->nm;
      W.m0 = ts->chain[0];
      W.m1 = ts->chain[1];
      W.m2 = ts->chain[2];
      for (int p = lane; p < n; p += TS) nxt[p] = cur[W.src_all(p)];
      if (lane == 0) {
        const int improved = bdd < 0.0;
        const int kk = ts->k;
        for (int s = 0; s < kk; ++s) {
          ts->usage[ts->sq[s]] += 1;
          ts->impr[ts->sq[s]] += improved;
        }
        ts->k_usage[kk - 1] += 1;
        ts->k_impr[kk - 1] += improved;
      }
      team_bar(team, TS);
      i16* t = cur;
      cur = nxt;
      nxt = t;
      phi = phi + bdd;
    }
    if (lane == 0) {
      A.rec_scal[(size_t)gi * A.P + ev] = phi;
      A.rec_pen[(size_t)gi * A.P + ev] = 0.0;
    }
    if (strictly_better(0.0, phi, bpen, bscal)) {  // team best-ever, first occurrence
      for (int p = lane; p < n; p += TS) A.best_genes[(size_t)ev * n + p] = cur[p];
      bscal = phi;
      bpen = 0.0;
      if (lane == 0) A.best_gen[ev] = g;
    }
  }

  // ---- write back ----------------------------------------------------------
  team_bar(team, TS);
  for (int p = lane; p < n; p += TS) A.genes[(size_t)ev * n + p] = cur[p];
  for (int i = lane; i < MAX_SEQ; i += TS) {
    A.usage[ev * MAX_SEQ + i] = ts->usage[i];
    A.impr[ev * MAX_SEQ + i] = ts->impr[i];
  }
  if (lane < 3) {
    A.k_usage[ev * 3 + lane] = ts->k_usage[lane];
    A.k_impr[ev * 3 + lane] = ts->k_impr[lane];
  }
  if (lane == 0) {
    A.scal[ev] = phi;
    A.pen[ev] = 0.0;
    A.best_scal[ev] = bscal;
    A.best_pen[ev] = bpen;
  }
  if (err) atomicOr(&A.gs->err, err);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    rd_pos += __shfl_xor_sync(0xffffffffu, rd_pos, off);
    rd_elem += __shfl_xor_sync(0xffffffffu, rd_elem, off);
  }
  if ((lane & 31) == 0) {
    atomicAdd(&A.gs->rd_pos, rd_pos);
    atomicAdd(&A.gs->rd_elem, rd_elem);
  }
}

}  // namespace go
