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
#include "go_perm_lns.cuh"

namespace go {

struct NoCustomOps {
  template <class Ctx>
  __device__ __forceinline__ static void run(int slot, Ctx& ctx) {
    ctx.err |= ERR_UNKNOWN_SEQ;
  }
};

template <class Acc>
struct TeamShared {  // (row kernels: go_evolve_row.cuh)
  Acc wd[32];
  int wl[32];
  Move chain[MAX_CHAIN];
  double bd;
  int nm, k, accept;
  int dnext;
  int sq[MAX_CHAIN];
  int usage[MAX_SEQ];
  int impr[MAX_SEQ];
  int k_usage[3];
  int k_impr[3];
  int nreq;
  int ndreq;
  int ngr;
  unsigned char cnt[16][MAX_SEQ];
};

// Team state of the permutation kernel; the per-warp arrays (argmin
// partials, lane-sort counts) follow it, sized by the team's warp count.
struct PermTeam {
  int accept;
  int dnext;                       // next deferred request to hand out (dynamic, per warp)
  int rnext;                       // next cooperative relocation / sampled-probe request
  int nreq;                        // pending cooperative relocations this step
  int ndreq;                       // pending deferred whole-row operators this step
  int ngr;                         // ... of which guided rebuilds (queued from the back)
  int pad;
  int usage[MAX_SEQ];
  int impr[MAX_SEQ];
  int k_usage[3];
  int k_impr[3];
};
template <class Acc>
struct PermWarpArrays {
  Acc* wd;               // [nw] warp argmin partials
  int* wl;               // [nw]
  unsigned char* cnt;    // [nw][MAX_SEQ] per-warp lane counts per sequence (lane sort)
  static __host__ __device__ unsigned bytes(int nw) {
    return (unsigned)(nw * (sizeof(Acc) + 4 + MAX_SEQ));
  }
  __device__ __forceinline__ void bind(unsigned char* p, int nw) {
    wd = (Acc*)p;
    wl = (int*)(p + nw * sizeof(Acc));
    cnt = p + nw * (sizeof(Acc) + 4);
  }
};

// Per logical lane state handed between threads across chain steps
// (structure of arrays after TeamShared; TS = lanes rounded up to 32).
template <class Acc>
struct LaneArrays {
  u64* mv;         // [3][TS] packed moves
  Acc* delta;      // [TS]
  u32* pos;        // [TS] stream words consumed
  u32* meta;       // [TS] k | nm | sq0 | sq1 | sq2
  unsigned short* order;  // [TS] thread slot -> logical lane
  unsigned short* req;    // [TS] lanes with a pending cooperative relocation
  unsigned short* dreq;   // [TS] lanes with a pending deferred whole-row operator
  static __host__ __device__ unsigned bytes(int TS) {
    return (unsigned)(TS * (3 * 8 + sizeof(Acc) + 4 + 4 + 2 + 2 + 2));
  }
  __device__ __forceinline__ void bind(unsigned char* p, int TS) {
    mv = (u64*)p;
    delta = (Acc*)(p + 3 * 8 * TS);
    pos = (u32*)(p + (3 * 8 + sizeof(Acc)) * TS);
    meta = pos + TS;
    order = (unsigned short*)(meta + TS);
    req = order + TS;
    dreq = req + TS;
  }
};

__device__ __forceinline__ u64 pack_move(const Move& m) { return pack_mv(m); }
__device__ __forceinline__ Move unpack_move(u64 v) { return unpack_mv(v); }
__device__ __forceinline__ u32 pack_meta(int k, int nm, int q0, int q1, int q2) {
  return (u32)k | ((u32)nm << 2) | ((u32)q0 << 4) | ((u32)q1 << 9) | ((u32)q2 << 14);
}
__device__ __forceinline__ int meta_k(u32 m) { return (int)(m & 3u); }
__device__ __forceinline__ int meta_nm(u32 m) { return (int)((m >> 2) & 3u); }
__device__ __forceinline__ int meta_sq(u32 m, int s) { return (int)((m >> (4 + 5 * s)) & 31u); }
// permutation kernel: the lane's chain base is its own materialised global row
// (bit 19) number `sel` (bit 20) instead of the team's current tour
enum : u32 { META_MAT = 1u << 19, META_SEL = 1u << 20, META_BASE = META_MAT | META_SEL };

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
    case SEQ_THREE_OPT: bi_three_opt(c); break;
    default:
      if (kind >= SEQ_CUSTOM_BASE) Custom::run(kind - SEQ_CUSTOM_BASE, c);
      else c.err |= ERR_UNKNOWN_SEQ;
  }
}

// Shared-memory carve-up common to the kernel and the host (engine.cu).
// Per team: [current row][PermTeam][per-warp arrays][LaneArrays]
// [per-warp scratch: row of n int16 + 32 ints].  Warp 0's scratch row doubles
// as the ping-pong row of the winner's apply (cur <-> nxt).
struct PermSmem {
  enum { WINTS = 32 };
  static __host__ __device__ unsigned align(unsigned x, unsigned a) { return (x + a - 1) / a * a; }
  static __host__ __device__ unsigned inst_off() { return 0; }
  static __host__ __device__ unsigned reg_off(unsigned inst_bytes) { return align(inst_bytes, 128); }
  static __host__ __device__ unsigned team_off(unsigned inst_bytes) {
    return reg_off(inst_bytes) + 768;
  }
  static __host__ __device__ unsigned row_bytes(int n) { return align(2u * n, 16); }
  static __host__ __device__ unsigned shared_off(int n) { return row_bytes(n); }
  template <class Acc>
  static __host__ __device__ unsigned warps_off(int n) {
    return align(shared_off(n) + (unsigned)sizeof(PermTeam), 16);
  }
  template <class Acc>
  static __host__ __device__ unsigned lanes_off(int n, int TS) {
    return align(warps_off<Acc>(n) + PermWarpArrays<Acc>::bytes(TS / 32), 16);
  }
  static __host__ __device__ unsigned scratch_bytes(int n) { return row_bytes(n) + 4 * WINTS; }
  template <class Acc>
  static __host__ __device__ unsigned scratch_off(int n, int TS) {
    return align(lanes_off<Acc>(n, TS) + LaneArrays<Acc>::bytes(TS), 16);
  }
  template <class Acc>
  static __host__ __device__ unsigned team_bytes(int n, int TS) {
    return align(scratch_off<Acc>(n, TS) + (unsigned)(TS / 32) * scratch_bytes(n), 16);
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
  double* s_cum = (double*)(sm + ro + 16);  // 32 doubles
  double* s_misc = s_cum + 32;               // kw[3], total
  int* s_kind = (int*)(s_misc + 4);          // 32 ints: implementation per registry index
  int* s_gord = s_kind + 32;                 // 32 ints: registry indices in sort order
  int* s_grank = s_gord + 32;                // 32 ints: sort position of a registry index
  if (A.inst_bytes) {
    stage_to_smem(sm, A.inst, A.inst_bytes, mbar);
    pol.d.m = (const typename decltype(pol.d)::Elem*)sm;
    pol.d.sbase = smem_u32(sm);
    pol.d.use_s = 1;
  }
  const RegistryDev* R = A.reg;
  const int nseq = R->nseq;
  for (int i = threadIdx.x; i < 32; i += blockDim.x) {
    s_cum[i] = R->cum[i];
    s_kind[i] = R->kind[i];
  }
  if (threadIdx.x < 3) s_misc[threadIdx.x] = R->kw[threadIdx.x];
  if (threadIdx.x == 3) s_misc[3] = R->total;
  if (threadIdx.x == blockDim.x - 1) {  // lane-sort order (any CTA size)
#ifdef GO_USER_OPS_FIRST
    // user operators first (long loops), then built-ins
    int j = 0;
    for (int pass = 0; pass < 2; ++pass)
      for (int i = 0; i < nseq; ++i)
        if ((R->kind[i] >= SEQ_CUSTOM_BASE) == (pass == 0)) {
          s_gord[j] = i;
          s_grank[i] = j++;
        }
#else
    // user operators (the long per-lane loops) spread evenly through the
    // built-ins, so consecutive warps do not both draw a long loop group: a
    // warp runs its lane groups one after another (SIMT), and the step waits
    // for its slowest warp
    int nu = 0;
    #pragma unroll 1
    for (int i = 0; i < nseq; ++i) nu += R->kind[i] >= SEQ_CUSTOM_BASE;
    const int nb = nseq - nu;
    int j = 0, bi = 0, ui = 0;
    for (int u = 0; u <= nu; ++u) {
      if (u < nu) {  // the next user operator
        while (R->kind[ui] < SEQ_CUSTOM_BASE) ++ui;
        s_gord[j] = ui;
        s_grank[ui] = j++;
        ++ui;
      }
      const int upto = nu ? (nb * (u + 1)) / nu : nb;  // built-ins between user operators
      while (bi < nseq && (j - (u + 1 < nu ? u + 1 : nu)) < upto) {
        if (R->kind[bi] < SEQ_CUSTOM_BASE) {
          s_gord[j] = bi;
          s_grank[bi] = j++;
        }
        ++bi;
      }
    }
    // the deferred whole-row sequences (no lane-execution work) right after the
    // first user operator: the warp holding that operator's long per-lane
    // loops gets as few other sequence groups as possible
    if (nu > 0) {
      int j2 = 0;
      s_grank[j2++] = s_gord[0];
      for (int pass = 0; pass < 2; ++pass)
        for (int i = 1; i < nseq; ++i)
          if (perm_deferred(R->kind[s_gord[i]]) == (pass == 0)) s_grank[j2++] = s_gord[i];
      for (int i = 0; i < nseq; ++i) s_gord[i] = s_grank[i];
      for (int i = 0; i < nseq; ++i) s_grank[s_gord[i]] = i;
    }
#endif
  }
  __syncthreads();

  const int TS = A.team_stride, T = A.T, n = A.n;
  const int team = threadIdx.x / TS, lane = threadIdx.x - team * TS;
  const int warp = lane >> 5, wl = lane & 31, nwarps = TS >> 5;
  const int ev = blockIdx.x * A.E + team;
  if (ev >= A.P) return;  // idle team slot; no CTA-wide barrier follows
  const long long evg = (long long)A.ev_offset + ev;

  unsigned char* tb = sm + PermSmem::team_off(A.inst_bytes) + team * A.team_smem;
  unsigned char* scr = tb + PermSmem::scratch_off<Acc>(n, TS);
  const unsigned scr_bytes = PermSmem::scratch_bytes(n);
  i16* cur = (i16*)tb;
  i16* nxt = (i16*)scr;  // warp 0's scratch row
  // this warp's shared-memory scratch (deferred whole-row operators)
  i16* const my_row = (i16*)(scr + warp * scr_bytes);  // warp 0: see nxt
  int* const my_int = (int*)(scr + warp * scr_bytes + PermSmem::row_bytes(n));
  PermTeam* ts = (PermTeam*)(tb + PermSmem::shared_off(n));
  PermWarpArrays<Acc> wa;
  wa.bind(tb + PermSmem::warps_off<Acc>(n), nwarps);
  LaneArrays<Acc> la;
  la.bind(tb + PermSmem::lanes_off<Acc>(n, TS), TS);

  #pragma unroll 1
  for (int p = lane; p < n; p += TS) cur[p] = A.genes[(size_t)ev * n + p];
  // lane-private global rows of deferred whole-row operators (2 per lane)
  i16* const lrow = A.lane_rows ? A.lane_rows + (size_t)ev * T * 2 * n : nullptr;
  auto lane_base = [&](int L, u32 meta) -> const i16* {
    return (meta & META_MAT) ? lrow + ((size_t)L * 2 + ((meta & META_SEL) ? 1 : 0)) * n : cur;
  };
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
    if (wl == 0) wa.wd[warp] = part;
    team_bar(team, TS);
    Acc tot = 0;
    for (int w = 0; w < nwarps; ++w) tot += wa.wd[w];
    phi = (double)tot;
    team_bar(team, TS);
  }
  double bscal = A.best_scal[ev], bpen = A.best_pen[ev];
  const double* kw = s_misc;
  const double total = s_misc[3];
  const unsigned lt_mask = (1u << wl) - 1u;
  int err = 0;
  unsigned long long rd_pos = 0, rd_elem = 0;

#ifdef GO_PHASE_TIMING
  unsigned long long prof[16] = {0}, t_last = clock64();
#define GO_TICK(slot) do { const unsigned long long t_ = clock64(); prof[(slot)] += t_ - t_last; t_last = t_; } while (0)
#else
#define GO_TICK(slot) do { } while (0)
#endif
  MateSel ms;
  int snap_min = (int)A.gen0;  // every team has published gen0 (host)
  for (int gi = 0; gi < A.ngen; ++gi) {
    const long long g = A.gen0 + gi;
    const double temp = A.temps[gi];
    // crossover snapshot of this generation (see EvolveArgs::snap)
    ms.init(A.snap, A.prog, (int)g, ev, A.P, A.islands, n);
#ifdef GO_PHASE_TIMING
    ms.prof = A.gs->prof;
#endif

    // ---- A: every lane draws k and its first sequence (identity mapping) ----
    if (lane < T) {
      Stream rng;
      rng.init(mix64_5_ool(A.seed, (u64)evg, (u64)g, (u64)lane, 0));
      const int k = sample_k(kw, rng);
      const int s0 = sample_seq(s_cum, nseq, total, rng);
      la.pos[lane] = rng.tell();
      la.meta[lane] = pack_meta(k, 0, s0, 0, 0);
      la.delta[lane] = (Acc)0;
    }
    // (no barrier: the step-0 ranking reads only this thread's own lane)

    // ---- B: chain steps.  Before each step the lanes are regrouped by
    //      sequence (counting sort over <= 31 ids) so a warp runs one
    //      operator at a time; deferred relocations are then resolved
    //      cooperatively by all warps of the team. ---------------------------
#pragma unroll 1
    for (int s = 0; s < MAX_CHAIN; ++s) {
      int hold_seq = 31;  // 31 = no work this step
      if (lane < T) {
        const u32 mt = la.meta[lane];
        if (meta_k(mt) > s) hold_seq = meta_sq(mt, s);
      }
      const unsigned grp = __match_any_sync(0xffffffffu, hold_seq);
      const int rank = __popc(grp & lt_mask);
      wa.cnt[warp * MAX_SEQ + wl] = 0;
      __syncwarp();
      if (hold_seq != 31 && rank == 0) wa.cnt[warp * MAX_SEQ + hold_seq] = (unsigned char)__popc(grp);
      team_bar(team, TS);
      GO_TICK(1 + 4 * s);
      if (lane == 0) {
        ts->nreq = 0;
        ts->ndreq = 0;
        ts->ngr = 0;
        ts->dnext = 0;
        ts->rnext = 0;
      }
      // exclusive scan of per-sequence totals in sort order (each warp redundantly)
      int tj = 0;
      if (wl < nseq) {
        const int q = s_gord[wl];
        #pragma unroll 1
        for (int w = 0; w < nwarps; ++w) tj += wa.cnt[w * MAX_SEQ + q];
      }
      int incl = tj;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, off);
        if (wl >= off) incl += v;
      }
      const int active = __shfl_sync(0xffffffffu, incl, 31);
      const int my_pos = hold_seq != 31 ? s_grank[hold_seq] : 0;
      int base = __shfl_sync(0xffffffffu, incl - tj, my_pos);
      if (hold_seq != 31) {
        #pragma unroll 1
        for (int w = 0; w < warp; ++w) base += wa.cnt[w * MAX_SEQ + hold_seq];
        la.order[base + rank] = (unsigned short)lane;
      }
      team_bar(team, TS);
      GO_TICK(2 + 4 * s);
      if (active == 0) break;  // uniform

#ifdef GO_PHASE_TIMING
      const unsigned long long t_ex0 = clock64();
#endif
      // the active lanes (sorted by sequence) in nwarps contiguous chunks, one per
      // warp: when fewer than TS lanes are active (later chain steps) every warp
      // gets a share instead of the first warps all of them (the step waits for
      // its slowest warp; a warp runs its sequence groups one after another)
      // Chunk c goes to warp (c + team) mod nwarps: a CTA's warp w runs on
      // scheduler w mod 4, so without the rotation every team's first chunk
      // (the long user-operator loops, sorted first) would share one scheduler
      const int chunk = min(32, (active + nwarps - 1) / nwarps);
      const int vwarp = (warp + nwarps - team % nwarps) % nwarps;
      const int pos = wl < chunk ? vwarp * chunk + wl : active;
      if (pos < active) {
        const int L = la.order[pos];
        Stream rng;
        rng.init(mix64_5_ool(A.seed, (u64)evg, (u64)g, (u64)L, 0));
        rng.seek(la.pos[L]);
        const u32 meta = la.meta[L];
        const int k = meta_k(meta);
        int nm = meta_nm(meta);
        int q0 = meta_sq(meta, 0), q1 = meta_sq(meta, 1), q2 = meta_sq(meta, 2);
        Chain C;
        C.reset(lane_base(L, meta), n);
        for (int i = 0; i < nm; ++i) C.push_packed(la.mv[i * TS + L]);
        Acc d = la.delta[L];
        PermCtx<Policy> c;
        c.rng = rng;
        c.L = C;
        c.pol = pol;
        c.err = 0;
        c.rd_pos = 0;
        c.rd_elem = 0;
        c.out.kind = MV_NONE;
        const int kind = s_kind[s == 0 ? q0 : (s == 1 ? q1 : q2)];
        bool pending = false;
        if (perm_deferred(kind)) {  // whole-row operator: resolved by a warp below
          // guided rebuilds (the longest) queue from the back and are handed out first
          if (kind == SEQ_GUIDED_REBUILD) la.dreq[TS - 1 - atomicAdd(&ts->ngr, 1)] = (unsigned short)L;
          else la.dreq[atomicAdd(&ts->ndreq, 1)] = (unsigned short)L;
          pending = true;
        } else {
          run_perm_op<Policy, Custom>(kind, c);
          rng = c.rng;
          if (c.out.kind == MV_RELOCATE_BEST) {
            la.mv[nm * TS + L] = pack_move(c.out);  // resolved below, nm unchanged
            la.req[atomicAdd(&ts->nreq, 1)] = (unsigned short)L;
            pending = true;
          } else if (c.out.kind != MV_NONE) {
            d += pol.delta(C, c.out, c.rd_pos, c.rd_elem);
            la.mv[nm * TS + L] = pack_move(c.out);
            ++nm;
          }
        }
        err |= c.err;
        rd_pos += c.rd_pos;
        rd_elem += c.rd_elem;
        if (!pending && s + 1 < k) {
          const int nq = sample_seq(s_cum, nseq, total, rng);
          if (s == 0) q1 = nq; else q2 = nq;
        }
        la.pos[L] = rng.tell();
        la.meta[L] = pack_meta(k, nm, q0, q1, q2) | (meta & META_BASE);
        la.delta[L] = d;
      }
#ifdef GO_PHASE_TIMING
      __syncwarp();  // slots 22.. : each warp's own lane-execution time, by warp index
      if (wl == 0 && warp < 4) atomicAdd(&A.gs->prof[22 + warp], clock64() - t_ex0);
      if (lane == 0) atomicAdd(&A.gs->prof[26], 1ull);
#endif
      team_bar(team, TS);
      GO_TICK(3 + 4 * s);

      // ---- cooperative best-slot relocations: one warp per request (32
      //      slots per step), handed out as warps free up
      const int nreq = ts->nreq;
      if (nreq > 0) {
#pragma unroll 1
        for (;;) {
          int r = 0;
          if (wl == 0) r = atomicAdd(&ts->rnext, 1);
          r = __shfl_sync(0xffffffffu, r, 0);
          if (r >= nreq) break;
          const int L = la.req[r];
          const u32 meta = la.meta[L];
          const int nm = meta_nm(meta);
          Chain C;
          const i16* bse = lane_base(L, meta);
          C.reset(bse, n);
          for (int i = 0; i < nm; ++i) C.push_packed(la.mv[i * TS + L]);
          const Move rq = unpack_move(la.mv[nm * TS + L]);
          const int st = rq.a, len = rq.b, m = n - len;
          const int f = C.at(st), l = C.at(st + len - 1);
          // slot p sits between rest[p-1] and rest[p] (rest = row without the
          // segment); 32 consecutive slots per step, prev / d(prev, f) come
          // from the neighbouring lane (d(prev, f) == d(f, prev) == previous
          // slot's d(l, next) when len == 1: TSP matrices are symmetric).
          // Scan is the narrowest exact type (int32 for int16 matrices); the
          // chain's moves are unpacked once and composed inline per slot.
          typedef typename Policy::Scan Scan;
          const Move c0 = unpack_mv(C.pm0), c1 = unpack_mv(C.pm1), c2 = unpack_mv(C.pm2);
          Scan best = 0;
          int bp = 0x7fffffff;
          int carry = C.at(m - 1 < st ? m - 1 : m - 1 + len);  // rest[m-1] = prev of slot 0
          Scan carry_b = pol.cost_scan(l, carry);
#pragma unroll 1
          for (int p0 = 0; p0 < m; p0 += 32) {
            const int p = p0 + wl;
            const bool in = p < m;
            int q = in ? (p < st ? p : p + len) : 0;
            if (nm > 2) q = move_src(c2, q);
            if (nm > 1) q = move_src(c1, q);
            if (nm > 0) q = move_src(c0, q);
            const int nxt = bse[q];
            const Scan b = pol.cost_scan(l, nxt);
            int prev = __shfl_up_sync(0xffffffffu, nxt, 1);
            Scan a_l = __shfl_up_sync(0xffffffffu, b, 1);
            if (wl == 0) {
              prev = carry;
              a_l = carry_b;
            }
            const Scan a = len == 1 ? a_l : pol.cost_scan(prev, f);
            const Scan c = pol.cost_scan(prev, nxt);
            const Scan dlt = Policy::kIntegral ? a + b - c : (Scan)(((double)a + (double)b) - (double)c);
            if (in && (bp == 0x7fffffff || dlt < best)) {  // p ascends per thread: first min
              best = dlt;
              bp = p;
            }
            carry = __shfl_sync(0xffffffffu, nxt, 31);
            carry_b = __shfl_sync(0xffffffffu, b, 31);
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            const Scan ob = __shfl_xor_sync(0xffffffffu, best, off);
            const int op = __shfl_xor_sync(0xffffffffu, bp, off);
            if (op != 0x7fffffff && (bp == 0x7fffffff || ob < best || (ob == best && op < bp))) {
              best = ob;
              bp = op;
            }
          }
          __syncwarp();  // every lane has read the request before lane 0 rewrites it
          if (wl == 0) {
            rd_pos += (unsigned)m + 3u;
            rd_elem += (len == 1 ? 2u : 3u) * (unsigned)m + 1u;
            Move mv;
            mv.kind = MV_SEGMENT;
            mv.a = st;
            mv.b = len;
            mv.c = bp;
            unsigned rp = 0, re = 0;
            const Acc d = la.delta[L] + pol.delta(C, mv, rp, re);
            la.mv[nm * TS + L] = pack_move(mv);
            const int k = meta_k(meta);
            int q1 = meta_sq(meta, 1), q2 = meta_sq(meta, 2);
            if (s + 1 < k) {  // continue the lane's stream after its operator's draws
              Stream rng;
              rng.init(mix64_5_ool(A.seed, (u64)evg, (u64)g, (u64)L, 0));
              rng.seek(la.pos[L]);
              const int nq = sample_seq(s_cum, nseq, total, rng);
              if (s == 0) q1 = nq; else q2 = nq;
              la.pos[L] = rng.tell();
            }
            la.meta[L] = pack_meta(k, nm + 1, meta_sq(meta, 0), q1, q2) | (meta & META_BASE);
            la.delta[L] = d;
          }
        }
        team_bar(team, TS);
        GO_TICK(4 + 4 * s);
      }

      // ---- deferred whole-row operators (go_perm_lns.cuh): one warp per lane
      const int ngr = ts->ngr, ndreq = ts->ndreq + ngr;
      if (ndreq > 0) {
#pragma unroll 1
        for (;;) {  // warps take requests as they free up (guided rebuilds, the longest, first)
          int r = 0;
          if (wl == 0) r = atomicAdd(&ts->dnext, 1);
          r = __shfl_sync(0xffffffffu, r, 0);
          if (r >= ndreq) break;
          const int L = r < ngr ? la.dreq[TS - 1 - r] : la.dreq[r - ngr];
          const u32 meta = la.meta[L];
          const int nm = meta_nm(meta), k = meta_k(meta);
          int q1 = meta_sq(meta, 1), q2 = meta_sq(meta, 2);
          const int kind = s_kind[meta_sq(meta, s)];
          Chain C;
          C.reset(lane_base(L, meta), n);
          for (int i = 0; i < nm; ++i) C.push_packed(la.mv[i * TS + L]);
          const int nsel = (meta & META_MAT) && !(meta & META_SEL) ? 1 : 0;
          i16* dst = lrow + ((size_t)L * 2 + nsel) * n;
          Stream rng;
          rng.init(mix64_5_ool(A.seed, (u64)evg, (u64)g, (u64)L, 0));
          rng.seek(la.pos[L]);
#ifdef GO_PHASE_TIMING
          const unsigned long long t_op = clock64();
#endif
          const DeferRes<Acc> dr = perm_defer(pol, C, kind, dst, warp == 0 ? nxt : my_row, my_int,
                                              rng, ms, n, wl);
          rng = dr.rng;
#ifdef GO_PHASE_TIMING
          if (wl == 0) {  // slots 16.. : (cycles, count) per deferred kind OX / shuffles / rebuild
            const int b = kind == SEQ_OX ? 16 : (kind == SEQ_GUIDED_REBUILD ? 20 : 18);
            atomicAdd(&A.gs->prof[b], clock64() - t_op);
            atomicAdd(&A.gs->prof[b + 1], 1ull);
          }
#endif
          Acc nd = la.delta[L];
          u32 bits = meta & META_BASE;
          int nm2 = nm;
          if (dr.changed) {
            nd = dr.len - (Acc)phi;
            bits = META_MAT | (nsel ? META_SEL : 0u);
            nm2 = 0;
          }
          __syncwarp();  // every lane has read la.pos / la.meta before lane 0 updates them
          if (wl == 0) {
            if (s + 1 < k) {
              const int nq = sample_seq(s_cum, nseq, total, rng);
              if (s == 0) q1 = nq; else q2 = nq;
            }
            la.pos[L] = rng.tell();
            la.meta[L] = pack_meta(k, nm2, meta_sq(meta, 0), q1, q2) | bits;
            la.delta[L] = nd;
            rd_pos += 2u * (unsigned)n;
            rd_elem += (unsigned)n;
          }
        }
        team_bar(team, TS);
        GO_TICK(15);
      }
    }

    // ---- C: team argmin over (delta, lane) -------------------------------------
    Acc bd = lane < T ? la.delta[lane] : AccMax<Acc>::value();  // padding lanes never win
    int bl = lane < T ? lane : 0x7fffffff;
    argmin_warp(bd, bl);
    if (wl == 0) {
      wa.wd[warp] = bd;
      wa.wl[warp] = bl;
    }
    team_bar(team, TS);
    GO_TICK(13);
    bd = wa.wd[0];
    bl = wa.wl[0];
    for (int w = 1; w < nwarps; ++w) {
      const Acc od = wa.wd[w];
      if (od < bd) {  // warps are in lane order: ties keep the lower lane
        bd = od;
        bl = wa.wl[w];
      }
    }
    const double bdd = (double)bd;
    if (lane == 0) {
      int acc = bdd < 0.0;
      if (!acc && temp > 0.0) {
        Stream ar;
        ar.init(mix64_5_ool(A.seed, (u64)evg, (u64)g, 0, 1));
        acc = ar.random() < exp(-bdd / temp);
      }
      ts->accept = acc;
      if (acc) {
        const u32 meta = la.meta[bl];
        const int kk = meta_k(meta);
        const int improved = bdd < 0.0;
        for (int s = 0; s < kk; ++s) {
          const int si = meta_sq(meta, s);
          ts->usage[si] += 1;
          ts->impr[si] += improved;
        }
        ts->k_usage[kk - 1] += 1;
        ts->k_impr[kk - 1] += improved;
      }
    }
    team_bar(team, TS);

    if (ts->accept) {
      Chain W;
      W.reset(lane_base(bl, la.meta[bl]), n);
      const int nm = meta_nm(la.meta[bl]);
      for (int i = 0; i < nm; ++i) W.push_packed(la.mv[i * TS + bl]);
      for (int p = lane; p < n; p += TS) nxt[p] = W.at(p);
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
    if (A.snap && gi + 1 < A.ngen)
      snap_publish(A.snap, A.prog, A.P, ev, n, (int)g + 1, cur, snap_min, lane, team, TS);
    if (strictly_better(0.0, phi, bpen, bscal) && !target_reached(A, bpen, bscal)) {  // team best-ever, first occurrence
      #pragma unroll 1
      for (int p = lane; p < n; p += TS) A.best_genes[(size_t)ev * n + p] = cur[p];
      bscal = phi;
      bpen = 0.0;
      if (lane == 0) A.best_gen[ev] = g;
    }
    GO_TICK(14);
  }

  // ---- write back ----------------------------------------------------------
  team_bar(team, TS);
#ifdef GO_PHASE_TIMING
  if (lane == 0)
    for (int i = 0; i < 16; ++i) atomicAdd(&A.gs->prof[i], prof[i]);
#endif
  #pragma unroll 1
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
  if (wl == 0) {
    atomicAdd(&A.gs->rd_pos, rd_pos);
    atomicAdd(&A.gs->rd_elem, rd_elem);
  }
}

}  // namespace go
