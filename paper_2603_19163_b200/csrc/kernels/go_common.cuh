// go_common.cuh — device primitives shared by every cuGenOpt kernel.
//
// No standard headers: this file is also compiled at run time by NVRTC when
// user operators are registered (paper §5.1 JIT pipeline).
//
//  * mix64          engine.py:74-83 (stream identity = the reference's hash)
//  * Philox4x32-10  counter-based words replacing MT19937
//  * Stream         CPython random.Random draw algorithms over those words:
//                   random() (two words, 53-bit), _randbelow (k = bit_length,
//                   rejection), so the draw ORDER is the reference's
//                   (oracle/rng.py WordRandom is the CPU twin)
//  * team barriers  one named barrier per evolver team (T lanes)
//  * bulk staging   cp.async.bulk (TMA 1-D) global -> shared with an mbarrier
#pragma once

namespace go {

typedef unsigned int u32;
typedef unsigned long long u64;
typedef long long i64;
typedef short i16;

enum { MAX_SEQ = 32, MAX_CHUNK = 64, MAX_CHAIN = 3 };

// sequence ids (operators.py:29-51)
enum SeqId {
  SEQ_SWAP = 0, SEQ_INSERT = 1, SEQ_REVERSE = 2, SEQ_OR_OPT = 3, SEQ_THREE_OPT = 4,
  SEQ_FLIP = 5, SEQ_SEG_FLIP = 6, SEQ_RANDOM_RESET = 7, SEQ_SEG_RESET = 8,
  SEQ_ROW_SWAP = 9, SEQ_ROW_SPLIT = 10, SEQ_ROW_MERGE = 11, SEQ_OX = 12,
  SEQ_UNIFORM_X = 13, SEQ_SEG_SHUFFLE = 14, SEQ_SCATTER_SHUFFLE = 15,
  SEQ_GUIDED_REBUILD = 16, SEQ_CUSTOM_BASE = 100
};

// sticky device error bits
enum ErrBits { ERR_OP_RANGE = 1, ERR_OP_MOVE = 2, ERR_UNKNOWN_SEQ = 4 };

__device__ __forceinline__ u64 mix64_fold(u64 h, u64 part) {
  h ^= part;
  h *= 0xBF58476D1CE4E5B9ull;
  h ^= h >> 27;
  h *= 0x94D049BB133111EBull;
  h ^= h >> 31;
  return h;
}

__device__ __forceinline__ u64 mix64_5(u64 a, u64 b, u64 c, u64 d, u64 e) {
  u64 h = 0x9E3779B97F4A7C15ull;
  h = mix64_fold(h, a);
  h = mix64_fold(h, b);
  h = mix64_fold(h, c);
  h = mix64_fold(h, d);
  return mix64_fold(h, e);
}

// one out-of-line copy for the permutation kernel, which keys lane streams at a
// dozen call sites (instruction-cache footprint); the row kernels inline it
__device__ __noinline__ u64 mix64_5_ool(u64 a, u64 b, u64 c, u64 d, u64 e) {
  return mix64_5(a, b, c, d, e);
}

__device__ __forceinline__ u64 mix64_3(u64 a, u64 b, u64 c) {
  u64 h = 0x9E3779B97F4A7C15ull;
  h = mix64_fold(h, a);
  h = mix64_fold(h, b);
  return mix64_fold(h, c);
}

// Philox4x32-10 block (Random123 constants); counter (c0,0,0,0), key (k0,k1)
__device__ __forceinline__ void philox_block(u32 c0, u32 k0, u32 k1, u32& o0, u32& o1, u32& o2,
                                             u32& o3) {
  u32 x0 = c0, x1 = 0, x2 = 0, x3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const u32 lo0 = 0xD2511F53u * x0, hi0 = __umulhi(0xD2511F53u, x0);
    const u32 lo1 = 0xCD9E8D57u * x2, hi1 = __umulhi(0xCD9E8D57u, x2);
    const u32 y0 = hi1 ^ x1 ^ k0, y2 = hi0 ^ x3 ^ k1;
    x0 = y0;
    x1 = lo1;
    x2 = y2;
    x3 = lo0;
  }
  o0 = x0;
  o1 = x1;
  o2 = x2;
  o3 = x3;
}

// One lane's stream: key = mix64(parts), words consumed w0..w3 per block.
// The Philox refill is kept out of line (by value, so the stream stays in
// registers): inlined at every draw site it made the evolve kernel several
// times larger than the instruction cache.
__device__ __noinline__ uint4 philox_refill(u32 c0, u32 k0, u32 k1) {
  uint4 w;
  philox_block(c0, k0, k1, w.x, w.y, w.z, w.w);
  return w;
}

// Counter-based access: word t of a stream is word t % 4 of Philox block t / 4,
// so draws at known word positions can be computed by any thread in parallel.
__device__ __forceinline__ u32 word_of(const uint4& w, u32 i) {
  return i == 0 ? w.x : (i == 1 ? w.y : (i == 2 ? w.z : w.w));
}
// random.Random.random() consuming words t, t+1
__device__ __forceinline__ double random_at(u32 k0, u32 k1, u32 t) {
  const uint4 w = philox_refill(t >> 2, k0, k1);
  const u32 a = word_of(w, t & 3);
  const u32 b = (t & 3) == 3 ? philox_refill((t >> 2) + 1, k0, k1).x : word_of(w, (t & 3) + 1);
  return ((double)(a >> 5) * 67108864.0 + (double)(b >> 6)) * (1.0 / 9007199254740992.0);
}

struct Stream {
  u32 k0, k1, ctr, w0, w1, w2, w3;
  int avail;

  __device__ __forceinline__ void init(u64 key) {
    k0 = (u32)key;
    k1 = (u32)(key >> 32);
    ctr = 0;
    avail = 0;
  }
  __device__ __forceinline__ u32 word() {
    if (avail == 0) refill();
    const u32 r = w0;
    w0 = w1;
    w1 = w2;
    w2 = w3;
    --avail;
    return r;
  }
  __device__ __forceinline__ void refill() {
    const uint4 w = philox_refill(ctr++, k0, k1);
    w0 = w.x;
    w1 = w.y;
    w2 = w.z;
    w3 = w.w;
    avail = 4;
  }
  // random.Random.random()
  __device__ __forceinline__ double random_inl() {
    const u32 a = word() >> 5;
    const u32 b = word() >> 6;
    return ((double)a * 67108864.0 + (double)b) * (1.0 / 9007199254740992.0);
  }
  // random.Random._randbelow_with_getrandbits, n > 0
  __device__ __forceinline__ int randbelow_inl(int n) {
    const int k = 32 - __clz(n);
    u32 r;
    do {
      r = word() >> (32 - k);
    } while (r >= (u32)n);
    return (int)r;
  }
  // The draws the operators call.  GO_OOL_DRAWS builds one out-of-line copy
  // each (stream passed and returned by value): 1.1k fewer instructions on C2
  // but measured 7 % slower (call and copy overhead on every draw), so the
  // default inlines them.
  __device__ __forceinline__ double random();
  __device__ __forceinline__ int randbelow(int n);
  __device__ __forceinline__ int randrange(int lo, int hi) { return lo + randbelow(hi - lo); }
  // words consumed so far / resume at a word position (lane state hand-off)
  __device__ __forceinline__ u32 tell() const { return ctr * 4u - (u32)avail; }
  __device__ __forceinline__ void seek(u32 pos) {
    ctr = pos >> 2;
    avail = 0;
    const int off = (int)(pos & 3u);
    if (off) {
      refill();
      for (int i = 0; i < off; ++i) word();
    }
  }
};

struct StreamInt {
  Stream s;
  int v;
};
struct StreamDbl {
  Stream s;
  double v;
};
__device__ __noinline__ StreamInt stream_randbelow(Stream s, int n) {
  StreamInt r;
  r.v = s.randbelow_inl(n);
  r.s = s;
  return r;
}
__device__ __noinline__ StreamDbl stream_random(Stream s) {
  StreamDbl r;
  r.v = s.random_inl();
  r.s = s;
  return r;
}
#ifdef GO_OOL_DRAWS
__device__ __forceinline__ int Stream::randbelow(int n) {
  const StreamInt r = stream_randbelow(*this, n);
  *this = r.s;
  return r.v;
}
__device__ __forceinline__ double Stream::random() {
  const StreamDbl r = stream_random(*this);
  *this = r.s;
  return r.v;
}
#else
__device__ __forceinline__ int Stream::randbelow(int n) { return randbelow_inl(n); }
__device__ __forceinline__ double Stream::random() { return random_inl(); }
#endif

// ---- CPython sampling helpers shared by the operator families ---------------
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

// random.sample(range(total), m) for m <= 30: CPython's pool method (a
// virtual pool of overrides in ovi/ovv, >= m entries each) when
// total <= setsize(m), else the set method
template <class C>
__device__ __forceinline__ void sample_range_buf(C& c, int total, int m, int* picks, int* ovi,
                                                 int* ovv) {
  if (total <= sample_setsize(m)) {
    int no = 0;
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
}

template <class C>
__device__ __forceinline__ void sample_range(C& c, int total, int m, int* picks) {
  int ovi[30], ovv[30];
  sample_range_buf(c, total, m, picks, ovi, ovv);
}

// sample(range(1, n), 3) sorted (operators.py:300).  Fixed-size loops, fully
// unrolled, so the pool overrides and picks stay in registers (dynamically
// indexed arrays would live in L2-backed local memory).
template <class C>
__device__ __forceinline__ void sample3_sorted(C& c, int n, int& i, int& j, int& k) {
  const int N = n - 1;  // population 1..n-1
  int out[3] = {0, 0, 0};
  if (N <= sample_setsize(3)) {  // pool method with a virtual pool
    int ovi[3] = {-1, -1, -1}, ovv[3] = {0, 0, 0};
    int no = 0;
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int jj = c.randbelow(N - t);
      int val = jj + 1;
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if (q < no && ovi[q] == jj) val = ovv[q];
      out[t] = val;
      // pool[jj] = pool[N - t - 1]
      const int src = N - t - 1;
      int sval = src + 1;
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if (q < no && ovi[q] == src) sval = ovv[q];
      bool found = false;
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if (q < no && ovi[q] == jj) {
          ovv[q] = sval;
          found = true;
        }
      if (!found) {
#pragma unroll
        for (int q = 0; q < 3; ++q)
          if (q == no) {
            ovi[q] = jj;
            ovv[q] = sval;
          }
        ++no;
      }
    }
  } else {  // set method
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      int jj;
      bool dup;
      do {
        jj = c.randbelow(N);
        dup = false;
#pragma unroll
        for (int q = 0; q < 3; ++q) dup |= (q < t && out[q] == jj + 1);
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

// ---- barriers -------------------------------------------------------------
__device__ __forceinline__ void team_bar(int team, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(nthreads) : "memory");
}

// ---- crossover snapshots: per-team progress instead of a grid barrier ---------
enum { SNAP_DEPTH = 8 };

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Polling loads: ld.acquire compiles to a strong load plus an L1 invalidation
// (CCTL.IVALL) of the whole SM, so spin loops poll with relaxed loads and
// acquire once, after the wait is over.
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// team: wait until every team has published generation >= target (one warp
// polls prog[0..P)), then publish this team's snapshot row of generation gnext
template <class G>
__device__ __forceinline__ void snap_publish(short* snap, int* prog, int P, int ev, int n,
                                             int gnext, const G* cur, int& gmin, int lane,
                                             int team, int nthreads) {
  const int target = gnext + 1 - SNAP_DEPTH;  // readers of the slot's old generation are done
  if (lane < 32 && target > gmin) {  // gmin: last observed minimum (progress only grows)
    for (;;) {
      int mn = 0x7fffffff;
      for (int t = lane; t < P; t += 32) {
        const int v = ld_relaxed(prog + t);
        mn = v < mn ? v : mn;
      }
      mn = (int)__reduce_min_sync(0xffffffffu, (unsigned)mn);
      gmin = mn;
      if (mn >= target) break;
      __nanosleep(256);
    }
    fence_acq_rel_gpu();  // pairs with the readers' st.release of their progress
  }
  team_bar(team, nthreads);
  short* dst = snap + ((size_t)(gnext % SNAP_DEPTH) * P + ev) * n;
#pragma unroll 1
  for (int p = lane; p < n; p += nthreads) dst[p] = (short)cur[p];
  team_bar(team, nthreads);
  if (lane == 0) {
    __threadfence();
    st_release(prog + ev, gnext);
  }
}

// Island membership of evolver `ev` among P (engine.py:790-798) and the mate
// draw of pick_mate (engine.py:553-559): None (no draw) for a 1-member island.
// The returned row is mate j's snapshot of generation `gen`, after waiting for
// team j to have published it.
struct MateSel {
  const short* rows;  // snapshot of this generation, [P][n]
  const int* prog;
  int start, size, pos, n, gen;
#ifdef GO_PHASE_TIMING
  unsigned long long* prof;  // GlobalState::prof (set by the kernel)
#endif
  __device__ __forceinline__ void init(const short* snap, const int* prog_, int g, int ev, int P,
                                       int islands, int n_) {
    rows = snap ? snap + (size_t)(g % SNAP_DEPTH) * P * n_ : nullptr;
    prog = prog_;
    gen = g;
    n = n_;
    const int base = P / islands, extra = P - base * islands;
    int isl;
    if (ev < extra * (base + 1)) {
      isl = ev / (base + 1);
      start = isl * (base + 1);
      size = base + 1;
    } else {
      isl = extra + (ev - extra * (base + 1)) / base;
      start = extra * (base + 1) + (isl - extra) * base;
      size = base;
    }
    pos = ev - start;
  }
  // the mate's evolver index (-1: none), after waiting for its snapshot
  template <class R>
  __device__ __forceinline__ int pick_index(R& rng) const {
    if (rows == nullptr || size <= 1) return -1;
    int j = rng.randbelow(size - 1);
    j += j >= pos;
    j += start;
    // one acquire load (pairs with the mate's st.release); if the mate is not
    // there yet, poll relaxed and acquire again once it is
    if (ld_acquire(prog + j) < gen) {
#ifdef GO_PHASE_TIMING
      const unsigned long long t0 = clock64();
#endif
      // exponential back-off: a waiting mate is typically tens of microseconds
      // behind, and every poll costs issue slots the SM's other warps could use
      unsigned ns = 128;
      while (ld_relaxed(prog + j) < gen) {
        __nanosleep(ns);
        ns = ns < 4096 ? ns * 2 : ns;
      }
      (void)ld_acquire(prog + j);
#ifdef GO_PHASE_TIMING
      atomicAdd(prof + 27, clock64() - t0);  // prof[27] cycles spent waiting, [28] waits
      atomicAdd(prof + 28, 1ull);
#endif
    }
#ifdef GO_PHASE_TIMING
    atomicAdd(prof + 29, 1ull);  // picks
#endif
    return j;
  }
  template <class R>
  __device__ __forceinline__ const short* pick(R& rng) const {
    const int j = pick_index(rng);
    return j < 0 ? nullptr : rows + (size_t)j * n;
  }
};

// ---- cp.async.bulk staging (global -> shared, one elected thread) ---------
__device__ __forceinline__ u32 smem_u32(const void* p) {
  return (u32)__cvta_generic_to_shared(p);
}

// Copies `bytes` (multiple of 16, both pointers 16B aligned) and waits.
// Must be called by every thread of the CTA (contains __syncthreads).
__device__ __forceinline__ void stage_to_smem(void* dst, const void* src, u32 bytes, u64* mbar) {
#ifndef GO_NO_BULK_COPY
  const u32 bar = smem_u32(mbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
    const u32 CH = 65536;
    for (u32 off = 0; off < bytes; off += CH) {
      const u32 sz = (bytes - off) < CH ? (bytes - off) : CH;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(smem_u32((char*)dst + off)), "l"((const char*)src + off), "r"(sz), "r"(bar)
          : "memory");
    }
  }
  __syncthreads();
  u32 done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(bar)
        : "memory");
  }
#else
  const int4* s = (const int4*)src;
  int4* d = (int4*)dst;
  for (u32 i = threadIdx.x; i < bytes / 16; i += blockDim.x) d[i] = __ldg(s + i);
  __syncthreads();
#endif
}

// ---- penalty-first comparison (core.py:315-347, Weighted mode) -----------
// returns true when (pa, sa) is strictly better than (pb, sb)
__device__ __forceinline__ bool strictly_better(double pa, double sa, double pb, double sb) {
  const bool fa = pa == 0.0, fb = pb == 0.0;
  if (fa != fb) return fa;
  if (!fa && pa != pb) return pa < pb;
  return sa < sb;
}
// compare(): -1 a better, 0 equal, 1 b better
__device__ __forceinline__ int compare3(double pa, double sa, double pb, double sb) {
  if (strictly_better(pa, sa, pb, sb)) return -1;
  if (strictly_better(pb, sb, pa, sa)) return 1;
  return 0;
}

// Multi-objective comparison (core.py:80-106, :315-347).  lex == 0: Weighted —
// solutions compare by (penalty, scal) where scal is the weighted scalarisation;
// lex == 1: Lexicographic over the objective vector in priority order
// (first, 1 - first) with per-objective tolerances.  Objectives here are
// routing "distance" / "vehicles" (builtins.py:80-152), both minimised.
struct MoCmp {
  int m;       // objectives (1 or 2)
  int lex;
  int first;   // priority_order[0]
  int maxmask; // bit i: objective i is Maximize (core.py:69-77)
  double tol[2];
};

// compare (core.py:315-347) for multi-objective runs: penalty first, then
// Weighted (scal) or Lexicographic over (o0, o1) in priority order with
// tolerances (|a - b| <= tol counts as a tie).  -1 a better, 0 equal, 1 b better.
__device__ __forceinline__ int compare_mo(double pa, double sa, double a0, double a1, double pb,
                                         double sb, double b0, double b1, const MoCmp& mo) {
  if (!mo.lex) return compare3(pa, sa, pb, sb);
  const bool fa = pa == 0.0, fb = pb == 0.0;
  if (fa != fb) return fa ? -1 : 1;
  if (!fa && pa != pb) return pa < pb ? -1 : 1;
  for (int k = 0; k < mo.m; ++k) {
    const int i = k == 0 ? mo.first : 1 - mo.first;
    const double x = i == 0 ? a0 : a1, y = i == 0 ? b0 : b1;
    if (fabs(__dsub_rn(x, y)) <= mo.tol[i]) continue;
    return (x < y) != ((mo.maxmask >> i & 1) != 0) ? -1 : 1;  // low wins unless Maximize
  }
  return 0;
}

// acceptance_delta, Lexicographic branch (engine.py:236-246): the difference on
// the first non-tied objective, plus pw * (penalty difference)
__device__ __forceinline__ double lex_delta(double c0, double c1, double cpen, double u0,
                                           double u1, double upen, double pw, const MoCmp& mo) {
  double d = 0.0;
  for (int k = 0; k < mo.m; ++k) {
    const int i = k == 0 ? mo.first : 1 - mo.first;
    const double diff = __dsub_rn(i == 0 ? c0 : c1, i == 0 ? u0 : u1);
    if (fabs(diff) <= mo.tol[i]) continue;
    d = (mo.maxmask >> i & 1) ? -diff : diff;
    break;
  }
  return __dadd_rn(d, __dmul_rn(pw, __dsub_rn(cpen, upen)));
}

__device__ __forceinline__ u64 globaltimer() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace go
