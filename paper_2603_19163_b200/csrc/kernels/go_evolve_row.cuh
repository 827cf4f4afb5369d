// go_evolve_row.cuh — evolve kernel for single-row problems evaluated on a
// materialised candidate: QAP (permutation), 0/1 knapsack (binary), JSP-int
// (integer priorities).  Same generation semantics as go_evolve_perm.cuh
// (engine.py:538-595); differences:
//   * every lane copies the current row into its own shared-memory row and
//     runs direct ports of the reference operators on it (go_row.cuh);
//   * lanes are regrouped by sequence before each chain step (warp = one
//     operator), as in the permutation kernel;
//   * evaluation is incremental over the touched position ranges:
//       QAP       delta over pairs (i, j) with i or j touched   (builtins.py:282-284)
//       knapsack  value / weight sums over touched cells        (builtins.py:258-262)
//       JSP-int   full serial-schedule decode per lane          (builtins.py:429-453)
//   * the winner's row is copied into the current row.
#pragma once
#include "go_args.cuh"
#include "go_common.cuh"
#include "go_dist.cuh"
#include "go_evolve_perm.cuh"
#include "go_part.cuh"
#include "go_row.cuh"

namespace go {

enum RowKind { RK_QAP = 0, RK_KNAP = 1, RK_JSP = 2, RK_PART = 3, RK_USER = 4 };

// Threads per CTA the statically built evolve kernel of a row kind is compiled
// for (__launch_bounds__(., 1)): 384 leaves 168 registers per thread (fewer
// spills into L2-backed local memory) and covers three teams of 128, the most
// the partition / JSP / knapsack BASELINE instances fit in shared memory; QAP
// (four teams of 128 fit) and the NVRTC user kernels keep 512.  choose_row()
// caps teams per CTA accordingly.
__host__ __device__ constexpr int row_max_threads(int kind) {
  return kind == RK_QAP || kind == RK_USER ? 512 : 384;
}
enum UserEnc { ENC_PERM = 0, ENC_BINARY = 1, ENC_INTEGER = 2 };

// ---- solution views handed to NVRTC-compiled user objectives ----------------------
// A user objective is `template <class Sol> double compute_obj(const Sol& sol,
// const Data& data)` reading genes as sol[i] (i < sol.n).  The views let trial
// evaluations run without copying the row.
template <class G>
struct RowSol {  // the row itself
  const G* r;
  int n;
  __device__ __forceinline__ int operator[](int i) const { return r[i]; }
  __device__ __forceinline__ int size() const { return n; }
};
template <class G>
struct OvSol {  // gene p replaced by v (binary / integer trials)
  const G* r;
  int n, p, v;
  __device__ __forceinline__ int operator[](int i) const { return i == p ? v : (int)r[i]; }
  __device__ __forceinline__ int size() const { return n; }
};
template <class G>
struct InsSol {  // v moved from slot q0 to slot pos of the row block [off, off + nb)
  const G* r;    // (permutation insertion trials; the block is the whole row, or one
  int n, off, nb, q0, pos, v;  // MULTI_FIXED row of the d1 x d2 solution)
  __device__ __forceinline__ int operator[](int i) const {
    const int b = i - off;
    if (b < 0 || b >= nb) return r[i];
    if (b == pos) return v;
    const int j = b < pos ? b : b - 1;  // index in the block without v
    return r[off + (j < q0 ? j : j + 1)];
  }
  __device__ __forceinline__ int size() const { return n; }
};

// lane / accept stream keys of the row kernels: out of line for the partition
// kernel (large, instruction-cache bound: C3 -14 % per chunk), inline for the
// others (QAP / knapsack: +4-8 % with a call per draw site)
template <int KIND>
__device__ __forceinline__ u64 row_key_k(u64 a, u64 b, u64 c, u64 d, u64 e) {
  return KIND == RK_PART ? mix64_5_ool(a, b, c, d, e) : mix64_5(a, b, c, d, e);
}

struct NoUser {  // built-in kinds: never called
  static constexpr bool kHasOps = false;  // user operator slots compiled in
  template <class S>
  __device__ __forceinline__ static double obj(const S&, const unsigned char*) { return 0.0; }
  template <class S>
  __device__ __forceinline__ static double pen(const S&, const unsigned char*) { return 0.0; }
  template <class S>
  __device__ __forceinline__ static double obj2(const S&, const unsigned char*) { return 0.0; }
  template <class C>
  __device__ __forceinline__ static void op(int, C& ctx, const unsigned char*) {
    ctx.err() |= ERR_UNKNOWN_SEQ;
  }
};


// scalar_fitness of a user solution view with one or two objectives
// (engine.py:215-222): Σ w_i·(±obj_i) from 0.0, then + pw·penalty
struct UserScore {
  const unsigned char* inst;
  double w, pw;
  int maximize;  // bit 0 / bit 1: objective 0 / 1 is Maximize
  double w2;
  int m;
  template <class U, class S>
  __device__ __forceinline__ double phi(const S& s) const {
    const double o0 = U::obj(s, inst);
    double sc = __dadd_rn(0.0, __dmul_rn(w, (maximize & 1) ? -o0 : o0));
    if (m == 2) {
      const double o1 = U::obj2(s, inst);
      sc = __dadd_rn(sc, __dmul_rn(w2, (maximize & 2) ? -o1 : o1));
    }
    return __dadd_rn(sc, __dmul_rn(pw, U::pen(s, inst)));
  }
};

// Instance data a user operator on a BUILT-IN row problem may read (the
// reference hands operators ctx.problem, whose arrays they index directly,
// e.g. demo_ops.py:18-21): QAP flow / distance, knapsack weights / values /
// capacity, JSP machine / duration per operation.  Out-of-range indices set
// the sticky error bit (the registration probe then excludes the operator).
enum { RI_NONE = 0, RI_QAP = 1, RI_KNAP = 2, RI_JSP = 3 };
struct RowInst {
  const unsigned char* b;  // instance image (shared or global memory)
  unsigned off1;           // second array (QAP D, knapsack v, JSP durations)
  int kind, elem, n;       // elem: QAP element bytes (2, 4) or 8 = float64
  double cap;
  int n_ops;               // JSP operations
  __device__ __forceinline__ double mat(unsigned off, int i, int j) const {
    const unsigned k = off + (unsigned)(i * n + j) * (unsigned)elem;
    return elem == 2 ? (double)*(const short*)(b + k)
                     : (elem == 4 ? (double)*(const int*)(b + k) : *(const double*)(b + k));
  }
};

// What a user operator snippet on a row problem sees as `ctx` (the reference's
// CustomOperator.apply(sol, rng, ctx), operators.py:79-88): the lane's candidate
// (d1 x d2 genes, row-major, flat index i < ctx.n), the lane stream with
// CPython's draw algorithms, Φ of the candidate (the `ctx.phi` the reference
// hands operators, engine.py:215-222) through the problem's own objective, and
// on built-in problems the instance arrays (RowInst).
template <class G, class U>
struct RowOpCtx {
  RowCtx<G>* c;
  UserScore us;
  int n, rows, width;  // flat genes, d1, d2
  RowInst in;          // kind RI_NONE on user (NVRTC-objective) problems
  __device__ __forceinline__ bool ok(int i, int lim) {
    const bool good = (unsigned)i < (unsigned)lim;
    c->err |= good ? 0 : ERR_OP_RANGE;
    return good;
  }
  __device__ __forceinline__ int get(int i) { return ok(i, n) ? (int)c->full[i] : 0; }
  __device__ __forceinline__ void set(int i, int v) {
    if (ok(i, n)) c->full[i] = (G)v;
  }
  __device__ __forceinline__ void swap(int i, int j) {
    if (!ok(i, n) || !ok(j, n)) return;
    const G t = c->full[i];
    c->full[i] = c->full[j];
    c->full[j] = t;
  }
  __device__ __forceinline__ int randbelow(int k) {
    if (k <= 0) { c->err |= ERR_OP_RANGE; return 0; }
    return c->rng.randbelow(k);
  }
  __device__ __forceinline__ int randrange(int a, int b) {
    if (b <= a) { c->err |= ERR_OP_RANGE; return a; }
    return c->rng.randrange(a, b);
  }
  __device__ __forceinline__ double random() { return c->rng.random(); }
  // QAP (builtins.py:265-290): flow F[i][j] between facilities, distance D[a][b]
  // between locations
  __device__ __forceinline__ double flow(int i, int j) {
    if (in.kind != RI_QAP || !ok(i, in.n) || !ok(j, in.n)) return 0.0;
    return in.mat(0, i, j);
  }
  __device__ __forceinline__ double dist(int a, int b) {
    if (in.kind != RI_QAP || !ok(a, in.n) || !ok(b, in.n)) return 0.0;
    return in.mat(in.off1, a, b);
  }
  // knapsack (builtins.py:240-262)
  __device__ __forceinline__ double weight(int i) {
    return in.kind == RI_KNAP && ok(i, in.n) ? ((const double*)in.b)[i] : 0.0;
  }
  __device__ __forceinline__ double value(int i) {
    return in.kind == RI_KNAP && ok(i, in.n) ? ((const double*)(in.b + in.off1))[i] : 0.0;
  }
  __device__ __forceinline__ double capacity() const { return in.cap; }
  // JSP-int (builtins.py:408-456): operation op = job * ops_per_job + k
  __device__ __forceinline__ int machine(int op) {
    return in.kind == RI_JSP && ok(op, in.n_ops) ? ((const int*)in.b)[op] : 0;
  }
  __device__ __forceinline__ int duration(int op) {
    return in.kind == RI_JSP && ok(op, in.n_ops) ? ((const int*)(in.b + in.off1))[op] : 0;
  }
  __device__ __forceinline__ double phi() {
    if (in.kind == RI_NONE) {
      const RowSol<G> s{c->full, n};
      return us.template phi<U>(s);
    }
    if (in.kind == RI_QAP) {  // Σ F_ij · D_{π_i π_j} (exact: products of integers)
      double t = 0.0;
      for (int i = 0; i < in.n; ++i)
        for (int j = 0; j < in.n; ++j)
          t += in.mat(0, i, j) * in.mat(in.off1, c->full[i], c->full[j]);
      return __dmul_rn(us.w, t);
    }
    if (in.kind == RI_KNAP) {  // Maximize value, penalty = weight over capacity
      double v = 0.0, w = 0.0;
      for (int i = 0; i < in.n; ++i) {
        v += value(i) * (double)c->full[i];
        w += weight(i) * (double)c->full[i];
      }
      const double over = __dsub_rn(w, in.cap);
      return __dadd_rn(__dmul_rn(us.w, -v), __dmul_rn(us.pw, over > 0.0 ? over : 0.0));
    }
    c->err |= ERR_OP_RANGE;  // JSP: the schedule decode is not offered to operators
    return 0.0;
  }
  __device__ __forceinline__ int& err() { return c->err; }
};

// What a user operator on a partition problem (VRPTW / CVRP, builtins.py:80-190)
// sees as `ctx`: routes (rows) of customer ids 0..n-1, a customer's matrix index
// is id + 1 with the depot at 0 (builtins.py:3-6, :122-123).  Moves keep the
// solution a partition; out-of-range arguments set the sticky error bit.
template <class U>
struct PartOpCtx {
  PartCtx* c;
  PartView pv;
  const RowArgs* X;
  double pw;
  int n, rows, width;  // customers, vehicles (d1), route capacity (d2)
  __device__ __forceinline__ bool ok(int i, int lim) {
    const bool good = (unsigned)i < (unsigned)lim;
    c->err |= good ? 0 : ERR_OP_RANGE;
    return good;
  }
  __device__ __forceinline__ int size(int r) { return ok(r, rows) ? (int)c->sz[r] : 0; }
  __device__ __forceinline__ int get(int r, int p) {
    if (!ok(r, rows) || !ok(p, c->sz[r])) return 0;
    return c->cells[c->start(r) + p];
  }
  // remove the customer at (r0, p0) and insert it at position p1 of route r1
  // (positions of the route after the removal, p1 <= its size)
  __device__ __forceinline__ void move(int r0, int p0, int r1, int p1) {
    if (!ok(r0, rows) || !ok(p0, c->sz[r0]) || !ok(r1, rows)) return;
    const int room = c->sz[r1] - (r1 == r0 ? 1 : 0);
    if ((unsigned)p1 > (unsigned)room || (r1 != r0 && c->sz[r1] >= width)) {
      c->err |= ERR_OP_MOVE;
      return;
    }
    const short v = c->remove(r0, p0);
    c->insert(r1, p1, v);
  }
  __device__ __forceinline__ void swap(int r0, int p0, int r1, int p1) {
    if (!ok(r0, rows) || !ok(p0, c->sz[r0]) || !ok(r1, rows) || !ok(p1, c->sz[r1])) return;
    const int a = c->start(r0) + p0, b = c->start(r1) + p1;
    const short t = c->cells[a];
    c->cells[a] = c->cells[b];
    c->cells[b] = t;
  }
  __device__ __forceinline__ void reverse(int r, int i, int j) {  // [i, j] of route r
    if (!ok(r, rows) || !ok(i, c->sz[r]) || !ok(j, c->sz[r]) || i > j) return;
    const int s = c->start(r);
    rev_short(c->cells + s, i, j);
  }
  // matrix distance between customers (-1 = the depot)
  __device__ __forceinline__ double dist(int a, int b) {
    if (!ok(a + 1, n + 1) || !ok(b + 1, n + 1)) return 0.0;
    return pv.dist[(a + 1) * (n + 1) + (b + 1)];
  }
  __device__ __forceinline__ double demand(int cst) { return ok(cst, n) ? pv.demand[cst] : 0.0; }
  __device__ __forceinline__ double ready(int cst) {
    return X->tw && ok(cst + 1, n + 1) ? pv.ready[cst + 1] : 0.0;
  }
  __device__ __forceinline__ double due(int cst) {
    return X->tw && ok(cst + 1, n + 1) ? pv.due[cst + 1] : 0.0;
  }
  __device__ __forceinline__ double service(int cst) {
    return X->tw && ok(cst + 1, n + 1) ? pv.service[cst + 1] : 0.0;
  }
  __device__ __forceinline__ double capacity() const { return X->capacity; }
  __device__ __forceinline__ int randbelow(int k) {
    if (k <= 0) { c->err |= ERR_OP_RANGE; return 0; }
    return c->rng.randbelow(k);
  }
  __device__ __forceinline__ int randrange(int a, int b) {
    if (b <= a) { c->err |= ERR_OP_RANGE; return a; }
    return c->rng.randrange(a, b);
  }
  __device__ __forceinline__ double random() { return c->rng.random(); }
  __device__ __forceinline__ double phi();  // defined after part_scal
  __device__ __forceinline__ int& err() { return c->err; }
};

// Instance views (all in shared memory once staged; `use_s` reads via ld.shared).
template <class E>
struct QapView {  // F then D, n x n each
  const E* f;
  const E* d;
  int n;
  unsigned fs, ds;
  int use_s;
  __device__ __forceinline__ typename AccOf<E>::T F(int i, int j) const {
    typedef typename AccOf<E>::T A;
    return use_s ? (A)LdShared<E>::load(fs + (unsigned)(i * n + j) * (unsigned)sizeof(E))
                 : (A)f[i * n + j];
  }
  __device__ __forceinline__ typename AccOf<E>::T D(int a, int b) const {
    typedef typename AccOf<E>::T A;
    return use_s ? (A)LdShared<E>::load(ds + (unsigned)(a * n + b) * (unsigned)sizeof(E))
                 : (A)d[a * n + b];
  }
  // the same with the instance's location fixed at compile time (hot loops are
  // instantiated for both, dispatched once on use_s)
  template <bool S>
  __device__ __forceinline__ typename AccOf<E>::T Fx(int i, int j) const {
    typedef typename AccOf<E>::T A;
    if constexpr (S) return (A)LdShared<E>::load(fs + (unsigned)(i * n + j) * (unsigned)sizeof(E));
    else return (A)f[i * n + j];
  }
  template <bool S>
  __device__ __forceinline__ typename AccOf<E>::T Dx(int a, int b) const {
    typedef typename AccOf<E>::T A;
    if constexpr (S) return (A)LdShared<E>::load(ds + (unsigned)(a * n + b) * (unsigned)sizeof(E));
    else return (A)d[a * n + b];
  }
};

struct KnapView {  // w[n], v[n] float64
  const double* w;
  const double* v;
  double cap;
};

struct JspView {  // per operation (job-major): machine, duration
  const int* mach;
  const int* dur;
  int n_jobs, per_job, n_mach;
};

struct RowLaneState {
  u32* pos;
  u32* meta;
  double* delta;
  double* nscal;
  double* npen;
  double* aux0;  // knapsack: new value sum
  double* aux1;  // knapsack: new weight sum
  unsigned short* order;
  unsigned char* nr;
  short* rlo;  // [MAX_RANGES][TS]
  short* rhi;
  unsigned short* greq;   // [TS] lanes with a deferred guided rebuild this step
  unsigned short* uxreq;  // [TS] lanes with a deferred uniform crossover this step
  static __host__ __device__ unsigned bytes(int TS) {
    return (unsigned)(TS * (4 + 4 + 8 * 5 + 2 + 1 + 4 * MAX_RANGES + 2 + 2) + 16);
  }
  __device__ __forceinline__ void bind(unsigned char* p, int TS) {
    delta = (double*)p;
    nscal = delta + TS;
    npen = nscal + TS;
    aux0 = npen + TS;
    aux1 = aux0 + TS;
    pos = (u32*)(aux1 + TS);
    meta = pos + TS;
    rlo = (short*)(meta + TS);
    rhi = rlo + MAX_RANGES * TS;
    order = (unsigned short*)(rhi + MAX_RANGES * TS);
    nr = (unsigned char*)(order + TS);
    greq = (unsigned short*)(nr + TS);
    uxreq = greq + TS;
  }
};

struct RowSmem {
  static __host__ __device__ unsigned align(unsigned x, unsigned a) { return (x + a - 1) / a * a; }
  // lane-row stride, 16-byte aligned (int4 row copies).  An odd number of
  // 4-byte words would spread the lanes' same-position reads over all 32 banks,
  // but its 4-byte copies measured slower overall (QAP +9 %, knapsack +5 %).
  static __host__ __device__ unsigned row_stride(int n, int gsize) { return align((unsigned)(n * gsize), 16); }
  // rows_smem: the T lane rows live in shared memory after the current row;
  // otherwise (long rows) they live in global memory (EvolveArgs::lane_rows)
  static __host__ __device__ unsigned team_bytes(int n, int gsize, int TS, int scratch_per_lane,
                                                 bool rows_smem = true) {
    return align(align(row_stride(n, gsize) * (rows_smem ? TS + 1 : 1), 16) + RowLaneState::bytes(TS) +
                     (unsigned)sizeof(TeamShared<double>) + (unsigned)(scratch_per_lane * TS),
                 16);
  }
};

// merge <= MAX_RANGES ranges into sorted disjoint ones; returns count (or -1: whole row)
__device__ __forceinline__ int merge_ranges(int nr, const short* lo_in, const short* hi_in, int n,
                                            int* lo, int* hi) {
  if (nr > MAX_RANGES) return -1;
  int m = 0;
  for (int i = 0; i < nr; ++i) {  // insertion by lo
    int a = lo_in[i], b = hi_in[i];
    int p = m;
    while (p > 0 && lo[p - 1] > a) {
      lo[p] = lo[p - 1];
      hi[p] = hi[p - 1];
      --p;
    }
    lo[p] = a;
    hi[p] = b;
    ++m;
  }
  int k = 0;
  for (int i = 0; i < m; ++i) {
    if (k > 0 && lo[i] <= hi[k - 1]) {
      if (hi[i] > hi[k - 1]) hi[k - 1] = hi[i];
    } else {
      lo[k] = lo[i];
      hi[k] = hi[i];
      ++k;
    }
  }
  (void)n;
  return k;
}

// ---- per-problem evaluation of a lane row against the current row -------------
template <class E, class G>
__device__ __forceinline__ double qap_delta(const QapView<E>& q, const G* cur, const G* row, int nm,
                                            const int* lo, const int* hi, unsigned& rd) {
  typedef typename AccOf<E>::T A;
  const int n = q.n;
  A d = 0;
  if (nm < 0) {  // whole row: Φ(row) - Φ(cur)
    for (int i = 0; i < n; ++i) {
      const int pi = row[i], ci = cur[i];
      for (int j = 0; j < n; ++j) d += q.F(i, j) * (q.D(pi, row[j]) - q.D(ci, cur[j]));
    }
    rd += 3u * (unsigned)(n * n);
    return (double)d;
  }
  // pairs with i touched.  The range loops stay rolled (lo / hi indexed from
  // local memory once per range): unrolled over MAX_RANGES they multiplied the
  // inner loops into half of the QAP kernel's instructions.
#pragma unroll 1
  for (int r = 0; r < nm; ++r)
    for (int i = lo[r]; i < hi[r]; ++i) {
      const int pi = row[i], ci = cur[i];
      for (int j = 0; j < n; ++j) d += q.F(i, j) * (q.D(pi, row[j]) - q.D(ci, cur[j]));
      rd += 3u * (unsigned)n;
    }
  // pairs with only j touched
  int gap_lo = 0;
#pragma unroll 1
  for (int r = 0; r <= nm; ++r) {
    const int gap_hi = r < nm ? lo[r] : n;
    for (int i = gap_lo; i < gap_hi; ++i) {
      const int ci = cur[i];
#pragma unroll 1
      for (int s = 0; s < nm; ++s)
        for (int j = lo[s]; j < hi[s]; ++j) d += q.F(i, j) * (q.D(ci, row[j]) - q.D(ci, cur[j]));
    }
    if (r < nm) gap_lo = hi[r];
  }
  return (double)d;
}

// Integer QAP: the lanes' deltas evaluated by the whole team.  A lane's delta is
// a sum of one term per touched position x (qap_delta's two parts regrouped:
// row x against every column, plus column x against every untouched row), each
// O(n); the team flattens the (lane, x) items, splits them evenly over its
// threads and accumulates in int64 shared-memory atomics.  Integer sums are
// order-free, so the deltas are bit-identical to qap_delta's; per-lane
// evaluation left 3/4 of every warp idle behind the lanes with the most touched
// positions (whole-row lanes cost n^2, a swap 4n).  Called by every thread of
// the team after each lane < T wrote its merged ranges (nr = 255: whole row) and
// touched count; acc / pre alias la.delta / la.nscal.
template <bool S, class E, class G>
__device__ __noinline__ void team_qap_delta_int(const QapView<E>& q, const G* cur,
                                                const unsigned char* rows, unsigned rs,
                                                const RowLaneState& la, int* wsum, int lane,
                                                int team, int TS) {
  typedef typename AccOf<E>::T A;
  const int n = q.n;
  auto F = [&](int x, int y) { return q.template Fx<S>(x, y); };
  auto D = [&](int x, int y) { return q.template Dx<S>(x, y); };
  int* pre = (int*)la.nscal;  // [TS] inclusive prefix of the touched counts
  unsigned long long* acc = (unsigned long long*)la.delta;
  const int warp = lane >> 5, wl = lane & 31, nwarps = TS >> 5;
  int c = pre[lane];  // the lane's count, replaced by its inclusive prefix
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, c, o);
    if (wl >= o) c += y;
  }
  if (wl == 31) wsum[warp] = c;
  team_bar(team, TS);
  for (int w = 0; w < warp; ++w) c += wsum[w];
  int total = 0;
  for (int w = 0; w < nwarps; ++w) total += wsum[w];
  pre[lane] = c;
  team_bar(team, TS);
#pragma unroll 1
  for (int it = lane; it < total; it += TS) {
    int a = 0, b = TS - 1;  // first L with pre[L] > it
    while (a < b) {
      const int m = (a + b) >> 1;
      if (pre[m] > it) b = m;
      else a = m + 1;
    }
    const int L = a;
    int x = it - (L > 0 ? pre[L - 1] : 0);
    const G* row = (const G*)(rows + (size_t)L * rs);
    const int nm = la.nr[L];
    A d = 0;
    if (nm == 255) {  // whole row: row x of sum F(i,j) (D(row_i,row_j) - D(cur_i,cur_j))
      const int pi = row[x], ci = cur[x];
      const int s0 = wl % n;  // rotated start: F row reads spread over the banks
#pragma unroll 4
      for (int j = s0; j < n; ++j) d += F(x, j) * (D(pi, row[j]) - D(ci, cur[j]));
#pragma unroll 4
      for (int j = 0; j < s0; ++j) d += F(x, j) * (D(pi, row[j]) - D(ci, cur[j]));
    } else {
      int r = 0;
#pragma unroll 1
      for (; r < nm; ++r) {
        const int len = la.rhi[r * TS + L] - la.rlo[r * TS + L];
        if (x < len) break;
        x -= len;
      }
      x += la.rlo[r * TS + L];
      const int pi = row[x], ci = cur[x];
      const int s0 = wl % n;
#pragma unroll 4
      for (int j = s0; j < n; ++j) d += F(x, j) * (D(pi, row[j]) - D(ci, cur[j]));
#pragma unroll 4
      for (int j = 0; j < s0; ++j) d += F(x, j) * (D(pi, row[j]) - D(ci, cur[j]));
      // column x against the untouched rows (the gaps between the ranges)
      const int rx = row[x], cx = cur[x];
      int gap_lo = 0;
#pragma unroll 1
      for (int g = 0; g <= nm; ++g) {
        const int gap_hi = g < nm ? la.rlo[g * TS + L] : n;
#pragma unroll 4
        for (int i = gap_lo; i < gap_hi; ++i) {
          const int ci2 = cur[i];
          d += F(i, x) * (D(ci2, rx) - D(ci2, cx));
        }
        if (g < nm) gap_lo = la.rhi[g * TS + L];
      }
    }
    atomicAdd(&acc[L], (unsigned long long)(long long)d);
  }
}

template <class G>
__device__ __forceinline__ void knap_delta(const KnapView& k, const G* cur, const G* row, int n,
                                           int nm, const int* lo, const int* hi, double& dv,
                                           double& dw) {
  dv = 0.0;
  dw = 0.0;
  if (nm < 0) {
    for (int p = 0; p < n; ++p) {
      const double x = (double)((int)row[p] - (int)cur[p]);
      if (x != 0.0) {
        dv += k.v[p] * x;
        dw += k.w[p] * x;
      }
    }
    return;
  }
#pragma unroll 1
  for (int r = 0; r < nm; ++r)
    for (int p = lo[r]; p < hi[r]; ++p) {
      const double x = (double)((int)row[p] - (int)cur[p]);
      if (x != 0.0) {
        dv += k.v[p] * x;
        dw += k.w[p] * x;
      }
    }
}

// serial schedule generator (builtins.py:429-453); scratch: job_free[n_jobs],
// mach_free[n_mach] (ints) then next[n_jobs] (bytes): jsp_scratch_ints() ints
// An odd count: the evaluation decodes one row per lane with every lane at the
// same offset of its own scratch at once, so an even stride (40 words for
// 20 x 15) put 8 lanes on each bank; an odd one gives 32 different banks.
__host__ __device__ __forceinline__ int jsp_scratch_ints(int n_jobs, int n_mach) {
  return (n_jobs + n_mach + (n_jobs + 3) / 4) | 1;
}
template <class G>
__device__ __forceinline__ int jsp_decode(const JspView& J, const G* prio, int* scratch) {
  int* jf = scratch;
  int* mf = jf + J.n_jobs;
  unsigned char* nxt = (unsigned char*)(mf + J.n_mach);
  for (int j = 0; j < J.n_jobs; ++j) {
    nxt[j] = 0;
    jf[j] = 0;
  }
  for (int m = 0; m < J.n_mach; ++m) mf[m] = 0;
  int span = 0;
  const int n_ops = J.n_jobs * J.per_job;
  for (int step = 0; step < n_ops; ++step) {
    int pick = -1, kp = 0, ko = 0;
    for (int j = 0; j < J.n_jobs; ++j) {
      const int k = nxt[j];
      if (k >= J.per_job) continue;
      const int op = j * J.per_job + k;
      const int pr = prio[op];
      if (pick < 0 || pr < kp || (pr == kp && op < ko)) {
        pick = j;
        kp = pr;
        ko = op;
      }
    }
    const int m = J.mach[ko], du = J.dur[ko];
    const int start = jf[pick] > mf[m] ? jf[pick] : mf[m];
    const int done = start + du;
    jf[pick] = done;
    mf[m] = done;
    nxt[pick] += 1;
    if (done > span) span = done;
  }
  return span;
}

// ---- op_guided_rebuild (operators.py:501-571) on a lane row ---------------------
// Every trial is scored with the run's scalar fitness (phi_fn, engine.py:548-550).
// QAP and JSP-int are integer-valued: QAP trial scores are exact int64 offsets
// (adjacent-swap deltas walking the value from the row end to position 0) and
// JSP scores are makespans, so first-minimum choices equal the reference's
// full re-evaluations.  Knapsack and partition scores are float64 in the
// reference's expression order (partitions: a full part_eval per trial).

// sorted descending (the single-row order of sorted(cells, key=(r, -p)))
__device__ __forceinline__ void sort_desc(int* a, int m) {
  for (int i = 1; i < m; ++i) {
    const int v = a[i];
    int j = i;
    while (j > 0 && a[j - 1] < v) {
      a[j] = a[j - 1];
      --j;
    }
    a[j] = v;
  }
}

template <class G>
__device__ __forceinline__ void row_pop(G* r, int size, int p) {
  for (int q = p; q < size - 1; ++q) r[q] = r[q + 1];
}

// QAP swap delta of positions (r, s) of permutation row (general F, D)
template <class E, class G>
__device__ __forceinline__ typename AccOf<E>::T qap_swap_delta(const QapView<E>& q, const G* row,
                                                               int n, int r, int s) {
  typedef typename AccOf<E>::T A;
  const int pr = row[r], ps = row[s];
  A d = (q.F(r, r) - q.F(s, s)) * (q.D(ps, ps) - q.D(pr, pr)) +
        (q.F(r, s) - q.F(s, r)) * (q.D(ps, pr) - q.D(pr, ps));
  for (int k = 0; k < n; ++k) {
    if (k == r || k == s) continue;
    const int pk = row[k];
    d += (q.F(r, k) - q.F(s, k)) * (q.D(ps, pk) - q.D(pr, pk)) +
         (q.F(k, r) - q.F(k, s)) * (q.D(pk, ps) - q.D(pk, pr));
  }
  return d;
}

// binary / integer: coordinate-greedy reset of a scatter of cells
template <int KIND, class G, class R>
__device__ __forceinline__ void gr_cells(const KnapView& kv, const JspView& jv, G* row, int n, int n_cfg, int lb,
                         int ub, double wobj, double pw, int* scratch, R& rng) {
  if (n == 0) return;
  const int ls = lns_scope(n_cfg);
  const int m = ls < n ? ls : n;
  int cells[30];
  sample_range(rng, n, m, cells);
  if (KIND == RK_KNAP) {
    lb = 0;
    ub = 1;
  }
  const int D = ub - lb + 1;
  int dom[16];
  int nd = D;
  if (D > 16) {  // sorted(rng.sample(domain, 16))
    sample_range(rng, D, 16, dom);
    for (int i = 1; i < 16; ++i) {
      const int v = dom[i];
      int j = i;
      while (j > 0 && dom[j - 1] > v) {
        dom[j] = dom[j - 1];
        --j;
      }
      dom[j] = v;
    }
    nd = 16;
    for (int i = 0; i < 16; ++i) dom[i] += lb;
  } else {
    for (int i = 0; i < D; ++i) dom[i] = lb + i;
  }
  double V = 0.0, W = 0.0;
  if (KIND == RK_KNAP)
    for (int p = 0; p < n; ++p) {
      const double x = (double)row[p];
      V += kv.v[p] * x;
      W += kv.w[p] * x;
    }
  for (int t = 0; t < m; ++t) {
    const int p = cells[t];
    const G old = row[p];
    int bv = (int)old;
    double bs = 0.0;
    bool have = false;
    for (int i = 0; i < nd; ++i) {
      const int v = dom[i];
      double sc;
      if (KIND == RK_KNAP) {
        const double dx = (double)(v - (int)old);
        const double nv = V + kv.v[p] * dx, nw = W + kv.w[p] * dx;
        const double over = __dsub_rn(nw, kv.cap);
        sc = __dadd_rn(__dadd_rn(0.0, __dmul_rn(wobj, -nv)), __dmul_rn(pw, over > 0.0 ? over : 0.0));
      } else {
        row[p] = (G)v;
        sc = (double)jsp_decode(jv, row, scratch);
      }
      if (!have || sc < bs) {
        have = true;
        bs = sc;
        bv = v;
      }
    }
    row[p] = (G)bv;
    if (KIND == RK_KNAP) {
      const double dx = (double)(bv - (int)old);
      V += kv.v[p] * dx;
      W += kv.w[p] * dx;
    }
  }
}

// ---- team-cooperative guided rebuild (QAP / JSP-int / partitions) --------------
// A lane that draws guided_rebuild is deferred; after the chain step the whole
// team resolves the deferred lanes one at a time.  Thread 0 replays the lane's
// stream (all of the operator's draws come first: cells, domain sample) and
// publishes them in `gx` (team scratch); the trials of each rebuilt value are
// then scored in parallel and the first minimum is applied.
struct GrShared {  // views into the team scratch (TeamShared::cnt, 128 ints)
  int* gx;
  __device__ __forceinline__ int& m() const { return gx[0]; }
  __device__ __forceinline__ int& nd() const { return gx[1]; }
  __device__ __forceinline__ int& res() const { return gx[2]; }
  __device__ __forceinline__ int& aux() const { return gx[3]; }
  __device__ __forceinline__ int& row() const { return gx[4]; }  // MULTI_FIXED home row
  __device__ __forceinline__ int* picks() const { return gx + 8; }   // [30]
  __device__ __forceinline__ int* taken() const { return gx + 40; }  // [30]
  __device__ __forceinline__ int* dom() const { return gx + 72; }    // [16]
  __device__ __forceinline__ int* score() const { return gx + 88; }  // [16] JSP makespans
};

// Thread 0: the draws of op_guided_rebuild for the lane (operators.py:501-571).
// `cells`: binary / integer encodings (coordinate-greedy branch).
template <int KIND>
__device__ __forceinline__ void gr_draw(Stream& rng, const GrShared& g, int n, int n_cfg, int lb,
                                        int ub, const short* sz, int d1, bool cells) {
  const int ls = lns_scope(n_cfg);
  int m = 0;
  if (cells) {
    if (n > 0) {
      m = ls < n ? ls : n;
      sample_range(rng, n, m, g.picks());
      const int D = ub - lb + 1;
      int nd = D;
      if (D > 16) {  // sorted(rng.sample(domain, 16))
        int* dm = g.dom();
        sample_range(rng, D, 16, dm);
        for (int i = 1; i < 16; ++i) {
          const int v = dm[i];
          int j = i;
          while (j > 0 && dm[j - 1] > v) {
            dm[j] = dm[j - 1];
            --j;
          }
          dm[j] = v;
        }
        nd = 16;
        for (int i = 0; i < 16; ++i) dm[i] += lb;
      } else {
        for (int i = 0; i < D; ++i) g.dom()[i] = lb + i;
      }
      g.nd() = nd;
    }
  } else if (n >= 3) {  // permutation cells (single row or partitions)
    m = ls < n - 1 ? ls : n - 1;
    int* pk = g.picks();
    sample_range(rng, n, m, pk);
    if (KIND != RK_PART) {  // sorted by (r, -p): descending positions
      for (int i = 1; i < m; ++i) {
        const int v = pk[i];
        int j = i;
        while (j > 0 && pk[j - 1] < v) {
          pk[j] = pk[j - 1];
          --j;
        }
        pk[j] = v;
      }
    } else {  // partitions: global cell -> (r, p), sorted by (r, -p), packed r << 16 | p
      for (int t = 0; t < m; ++t) {
        int gi = pk[t], r = 0;
        while (gi >= sz[r]) {
          gi -= sz[r];
          ++r;
        }
        pk[t] = (r << 16) | (0xFFFF - gi);  // ascending key == (r asc, p desc)
      }
      for (int i = 1; i < m; ++i) {
        const int v = pk[i];
        int j = i;
        while (j > 0 && pk[j - 1] > v) {
          pk[j] = pk[j - 1];
          --j;
        }
        pk[j] = v;
      }
      for (int t = 0; t < m; ++t) pk[t] = (pk[t] & 0xFFFF0000) | (0xFFFF - (pk[t] & 0xFFFF));
    }
  }
  g.m() = m;
  (void)d1;
}

// QAP swap delta of positions (a, a+1) in the row r (size n-1, without v) with v
// inserted at a+1 (= the walk step moving v from a+1 to a).  r(k) is virtual:
// r[k] = row[k < q0 ? k : k + 1] (row still holds v at q0).
template <bool S, class E, class G>
__device__ __forceinline__ typename AccOf<E>::T qap_walk_delta(const QapView<E>& q, const G* row,
                                                               int n, int q0, int v, int a) {
  typedef typename AccOf<E>::T A;
  auto F = [&](int x, int y) { return q.template Fx<S>(x, y); };
  auto D = [&](int x, int y) { return q.template Dx<S>(x, y); };
  const int b = a + 1;
  auto rr = [&](int k) -> int { return row[k < q0 ? k : k + 1]; };
  const int pa = rr(a), pb = v;  // before the swap: r[a] at a, v at b
  A d = (F(a, a) - F(b, b)) * (D(pb, pb) - D(pa, pa)) +
        (F(a, b) - F(b, a)) * (D(pb, pa) - D(pa, pb));
  for (int k = 0; k < n; ++k) {
    if (k == a || k == b) continue;
    const int pk = rr(k < a ? k : k - 1);
    d += (F(a, k) - F(b, k)) * (D(pb, pk) - D(pa, pk)) +
         (F(k, a) - F(k, b)) * (D(pk, pb) - D(pk, pa));
  }
  return d;
}

// rewrite row so that element at old position `src(t)` lands at t (team, two phases)
template <class G, class F>
__device__ __forceinline__ void team_permute(G* row, int n, const F& src, int lane, int team,
                                             int TS) {
  G v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int t = lane + i * TS;
    if (t < n) v[i] = row[src(t)];
  }
  team_bar(team, TS);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int t = lane + i * TS;
    if (t < n) row[t] = v[i];
  }
  team_bar(team, TS);
}

// pop the picks (descending positions) and park them at the row end in pick
// order (operators.py:527-533); taken values published in g.taken()
template <class G>
__device__ void team_pop_park(G* row, int n, const GrShared& g, int lane, int team, int TS) {
  const int m = g.m();
  const int* pk = g.picks();
  if (lane == 0)
    for (int t = 0; t < m; ++t) g.taken()[t] = row[pk[t]];
  if (n > 8 * TS) {  // rows longer than the register staging: serial moves by thread 0
    if (lane == 0) {
      int size = n;
      for (int t = 0; t < m; ++t) {
        row_pop(row, size, pk[t]);
        --size;
      }
      for (int t = 0; t < m; ++t) row[size++] = (G)g.taken()[t];
    }
    team_bar(team, TS);
  } else {
    team_permute(row, n, [&](int t) -> int {
      if (t >= n - m) return pk[t - (n - m)];
      int p = t;  // t-th survivor: skip picked positions in ascending order
      for (int j = m - 1; j >= 0; --j) p += pk[j] <= p;
      return p;
    }, lane, team, TS);
  }
}

// move the value at slot q0 to slot b (the row keeps n slots)
template <class G>
__device__ void team_move(G* row, int n, int q0, int b, int v, int lane, int team, int TS) {
  if (n > 8 * TS) {
    if (lane == 0) {
      row_pop(row, n, q0);
      for (int p = n - 1; p > b; --p) row[p] = row[p - 1];
      row[b] = (G)v;
    }
    team_bar(team, TS);
  } else {
    team_permute(row, n, [&](int x) -> int {
      if (x == b) return q0;
      const int r = x < b ? x : x - 1;  // index in the row without v
      return r < q0 ? r : r + 1;
    }, lane, team, TS);
  }
}

template <class E, class G>
__device__ void team_gr_qap(const QapView<E>& q, G* row, int n, const GrShared& g, double* sbuf,
                            int lane, int team, int TS) {
  typedef typename AccOf<E>::T A;
  const int m = g.m();
  if (m == 0) return;
  team_pop_park(row, n, g, lane, team, TS);
  for (int t = 0; t < m; ++t) {
    const int v = g.taken()[t];
    for (int p = lane; p < n; p += TS)
      if (row[p] == v) g.res() = p;
    team_bar(team, TS);
    const int q0 = g.res();
    // walk v from n-1 down to 0: sd[a] = delta of the step a+1 -> a, computed in
    // parallel chunks of `cap` steps; thread 0 accumulates the scores (relative
    // to v at n-1) from the top, lower positions winning ties
    A* sd = (A*)sbuf;
    const int cap = 5 * TS;
    A sc = 0, best = 0;
    int bp = n - 1;
    for (int hi = n - 1; hi > 0; hi -= cap) {
      const int lo = hi - cap > 0 ? hi - cap : 0;
      for (int a = lo + lane; a < hi; a += TS)
        sd[a - lo] = q.use_s ? qap_walk_delta<true>(q, row, n, q0, v, a)
                             : qap_walk_delta<false>(q, row, n, q0, v, a);
      team_bar(team, TS);
      if (lane == 0)
        for (int a = hi - 1; a >= lo; --a) {
          sc += sd[a - lo];
          if (sc <= best) {
            best = sc;
            bp = a;
          }
        }
      team_bar(team, TS);
    }
    if (lane == 0) g.aux() = bp;
    team_bar(team, TS);
    team_move(row, n, q0, g.aux(), v, lane, team, TS);
  }
}

// user objectives: guided rebuild trials scored by the NVRTC-compiled objective
// on virtual rows (no copies), in parallel over the team

template <class U, class G>
__device__ void team_gr_user_perm(G* full, int ntot, int off, int n, const GrShared& g,
                                  const UserScore& us, double* sbuf, TeamShared<double>* ts,
                                  int lane, int team, int TS) {
  const int m = g.m();
  if (m == 0) return;
  G* row = full + off;  // the rebuilt row; trials are scored on the whole solution
  const int warp = lane >> 5, wl = lane & 31, nwarps = TS >> 5;
  team_pop_park(row, n, g, lane, team, TS);
  for (int t = 0; t < m; ++t) {
    const int v = g.taken()[t];
    for (int p = lane; p < n; p += TS)
      if (row[p] == v) g.res() = p;
    team_bar(team, TS);
    const int q0 = g.res();
    double bs = 0.0;
    int bi = 0x7fffffff;
    for (int pos = lane; pos < n; pos += TS) {  // ascending per thread: first minimum
      const InsSol<G> sol{full, ntot, off, n, q0, pos, v};
      const double sc = us.template phi<U>(sol);
      if (bi == 0x7fffffff || sc < bs) {
        bs = sc;
        bi = pos;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, bs, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (oi != 0x7fffffff && (bi == 0x7fffffff || ob < bs || (ob == bs && oi < bi))) {
        bs = ob;
        bi = oi;
      }
    }
    if (wl == 0) {
      sbuf[warp] = bs;
      ts->wl[warp] = bi;
    }
    team_bar(team, TS);
    if (lane == 0) {
      double b = 0.0;
      int ib = 0x7fffffff;
      for (int w = 0; w < nwarps; ++w) {
        const int oi = ts->wl[w];
        if (oi != 0x7fffffff && (ib == 0x7fffffff || sbuf[w] < b || (sbuf[w] == b && oi < ib))) {
          b = sbuf[w];
          ib = oi;
        }
      }
      g.aux() = ib;
    }
    team_bar(team, TS);
    team_move(row, n, q0, g.aux(), v, lane, team, TS);
  }
}

template <class U, class G>
__device__ void team_gr_user_cells(G* row, int n, const GrShared& g, const UserScore& us,
                                   double* sbuf, int lane, int team, int TS) {
  const int m = g.m(), nd = g.nd();
  for (int t = 0; t < m; ++t) {
    const int p = g.picks()[t];
    for (int i = lane; i < nd; i += TS) {
      const OvSol<G> sol{row, n, p, g.dom()[i]};
      sbuf[i] = us.template phi<U>(sol);
    }
    team_bar(team, TS);
    if (lane == 0) {  // first minimum in domain order
      int bi = 0;
      for (int i = 1; i < nd; ++i)
        if (sbuf[i] < sbuf[bi]) bi = i;
      row[p] = (G)g.dom()[bi];
    }
    team_bar(team, TS);
  }
}

// warp-cooperative serial schedule generator (builtins.py:429-453) with one
// priority overridden (position ovp := ovv); lanes own jobs wl + 32 s.
// Fast path (n_jobs, n_machines <= 32, <= 255 operations per job): lane j owns
// job j and machine j in registers; key = (priority, job, index) orders exactly
// like (priority, op) since op = job * per_job + index.
// Warp-cooperative decode state (lane j owns job j and machine j).
struct JspWarp {
  int nx, jf, mfr, pr, pn, span, step;  // pn: priority of the op after the head
  int mh, dh, mh2, dh2;                 // machine / duration of the head op and of the next
};

// Runs steps of the fast-path decode from `st` until every operation is
// scheduled, or (stop_job >= 0) until job stop_job's next operation index
// becomes stop_k (that operation is then a candidate and its priority matters).
// Priority of operation ovp is ovv.  Every lane computes the completion time its
// head operation would have if chosen (its job's finish vs its machine's, read
// from the machine's lane) while the warp reduces the keys, so a step is one
// min-reduction and one shuffle of the winner's time instead of reduction ->
// operation load -> two shuffles; machines and durations of each job's next
// two operations are prefetched into registers.
template <class G>
__device__ __forceinline__ void jsp_warp_run(const JspView& J, const G* prio, int ovp, int ovv,
                                             int wl, JspWarp& st, int stop_job, int stop_k) {
  const int pj = J.per_job;
  const bool mine = wl < J.n_jobs;
  const int n_ops = J.n_jobs * pj;
  for (; st.step < n_ops; ++st.step) {
    if (stop_job >= 0 && __shfl_sync(0xffffffffu, st.nx, stop_job) == stop_k) return;
    const bool live = mine && st.nx < pj;
    const unsigned key = live ? ((unsigned)st.pr << 16) | ((unsigned)wl << 8) | (unsigned)st.nx
                              : 0xFFFFFFFFu;
    const int mfm = __shfl_sync(0xffffffffu, st.mfr, st.mh & 31);
    const int cand = (st.jf > mfm ? st.jf : mfm) + st.dh;
    const unsigned kmin = __reduce_min_sync(0xffffffffu, key);
    const int j = (int)((kmin >> 8) & 0xFFu);
    const int done = __shfl_sync(0xffffffffu, cand, j);
    const int m = __shfl_sync(0xffffffffu, st.mh, j);
    if (wl == m) st.mfr = done;
    if (wl == j) {
      st.jf = done;
      ++st.nx;
      st.pr = st.pn;  // prefetched priority of the new head
      st.mh = st.mh2;
      st.dh = st.dh2;
      const int o2 = j * pj + st.nx + 1;  // and the one after it, off the critical path
      if (st.nx + 1 < pj) {
        st.pn = o2 == ovp ? ovv : (int)prio[o2];
        st.mh2 = J.mach[o2];
        st.dh2 = J.dur[o2];
      }
    }
    st.span = done > st.span ? done : st.span;
  }
}

// K guided-rebuild trials of one warp decoded together: the trials share the
// prefix `st[k]` starts from and differ only in the priority of an operation that
// is already a job head, so every later prefetch reads the row itself.  The K
// step bodies are independent dependency chains (shuffle -> min-reduce ->
// shuffles), interleaved by the unrolled loop to hide their latency; updates are
// selects, not branches, so the scheduler can mix them.
template <int K, class G>
__device__ __forceinline__ void jsp_warp_run_k(const JspView& J, const G* prio, int wl,
                                               JspWarp (&st)[K]) {
  const int pj = J.per_job;
  const bool mine = wl < J.n_jobs;
  const int n_ops = J.n_jobs * pj;
#pragma unroll 1
  for (int step = st[0].step; step < n_ops; ++step) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      JspWarp& w = st[k];
      const bool live = mine && w.nx < pj;
      const unsigned key = live ? ((unsigned)w.pr << 16) | ((unsigned)wl << 8) | (unsigned)w.nx
                                : 0xFFFFFFFFu;
      const int mfm = __shfl_sync(0xffffffffu, w.mfr, w.mh & 31);
      const int cand = (w.jf > mfm ? w.jf : mfm) + w.dh;
      const unsigned kmin = __reduce_min_sync(0xffffffffu, key);
      const int j = (int)((kmin >> 8) & 0xFFu);
      const int done = __shfl_sync(0xffffffffu, cand, j);
      const int m = __shfl_sync(0xffffffffu, w.mh, j);
      w.mfr = wl == m ? done : w.mfr;
      const bool me = wl == j;
      w.jf = me ? done : w.jf;
      w.nx += me ? 1 : 0;
      w.pr = me ? w.pn : w.pr;
      w.mh = me ? w.mh2 : w.mh;
      w.dh = me ? w.dh2 : w.dh;
      if (me && w.nx + 1 < pj) {
        const int o2 = j * pj + w.nx + 1;
        w.pn = (int)prio[o2];
        w.mh2 = J.mach[o2];
        w.dh2 = J.dur[o2];
      }
      w.span = done > w.span ? done : w.span;
    }
  }
}

template <class G>
__device__ __forceinline__ JspWarp jsp_warp_start(const JspView& J, const G* prio, int ovp,
                                                  int ovv, int wl) {
  JspWarp st;
  st.nx = st.jf = st.mfr = st.span = st.step = 0;
  st.mh = st.dh = st.mh2 = st.dh2 = 0;
  const int op0 = wl * J.per_job;
  st.pr = wl < J.n_jobs ? (op0 == ovp ? ovv : (int)prio[op0]) : 0;
  st.pn = wl < J.n_jobs && J.per_job > 1 ? (op0 + 1 == ovp ? ovv : (int)prio[op0 + 1]) : 0;
  if (wl < J.n_jobs) {
    st.mh = J.mach[op0];
    st.dh = J.dur[op0];
    if (J.per_job > 1) {
      st.mh2 = J.mach[op0 + 1];
      st.dh2 = J.dur[op0 + 1];
    }
  }
  return st;
}

// Fast path (n_jobs, n_machines <= 32, <= 255 operations per job): lane j owns
// job j and machine j in registers; key = (priority, job, index) orders exactly
// like (priority, op) since op = job * per_job + index.
template <class G>
__device__ __forceinline__ int jsp_decode_warp32(const JspView& J, const G* prio, int ovp, int ovv,
                                                 int wl) {
  JspWarp st = jsp_warp_start(J, prio, ovp, ovv, wl);
  jsp_warp_run(J, prio, ovp, ovv, wl, st, -1, 0);
  return st.span;
}

template <class G>
__device__ __forceinline__ int jsp_decode_warp(const JspView& J, const G* prio, int ovp, int ovv,
                                               int* mf, int wl) {
  if (J.n_jobs <= 32 && J.n_mach <= 32 && J.per_job < 256 && J.n_jobs * J.per_job < 32768)
    return jsp_decode_warp32(J, prio, ovp, ovv, wl);
  int nx[4], jf[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    nx[s] = 0;
    jf[s] = 0;
  }
  for (int m = wl; m < J.n_mach; m += 32) mf[m] = 0;
  __syncwarp();
  int span = 0;
  const int n_ops = J.n_jobs * J.per_job;
  for (int step = 0; step < n_ops; ++step) {
    unsigned key = 0xFFFFFFFFu;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int j = wl + 32 * s;
      if (j < J.n_jobs && nx[s] < J.per_job) {
        const int op = j * J.per_job + nx[s];
        const int pr = op == ovp ? ovv : (int)prio[op];
        const unsigned k2 = ((unsigned)pr << 16) | (unsigned)op;
        key = k2 < key ? k2 : key;
      }
    }
    key = __reduce_min_sync(0xFFFFFFFFu, key);
    const int op = (int)(key & 0xFFFFu);
    const int j = op / J.per_job;
    if ((j & 31) == wl) {
      const int s = j >> 5;
      const int m = J.mach[op];
      int jfs = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) jfs = t == s ? jf[t] : jfs;
      const int mfm = mf[m];
      const int done = (jfs > mfm ? jfs : mfm) + J.dur[op];
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (t == s) {
          jf[t] = done;
          nx[t] += 1;
        }
      mf[m] = done;
      span = done > span ? done : span;
    }
    __syncwarp();
  }
  return __reduce_max_sync(0xFFFFFFFFu, (unsigned)span);
}

template <int K, class G>
__device__ __forceinline__ void jsp_gr_trials(const JspView& J, const G* row, const GrShared& g,
                                              const JspWarp& base, int jp, int kp, int nd,
                                              int warp, int nwarps, int wl) {
#pragma unroll 1
  for (int i0 = warp * K; i0 < nd; i0 += nwarps * K) {
    JspWarp st[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      st[k] = base;
      const int v = g.dom()[i0 + k < nd ? i0 + k : nd - 1];
      if (wl == jp && st[k].nx == kp) st[k].pr = v;  // op p is job jp's head: its trial priority
    }
    jsp_warp_run_k<K>(J, row, wl, st);
    if (wl == 0) {
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (i0 + k < nd) g.score()[i0 + k] = st[k].span;
    }
  }
}

template <class G>
__device__ void team_gr_jsp(const JspView& J, G* row, const GrShared& g, int* scratch,
                            int scratch_ints, int lane, int team, int TS) {
  const int m = g.m(), nd = g.nd();
  const int warp = lane >> 5, wl = lane & 31, nwarps = TS >> 5;
  int* mf = scratch + warp * scratch_ints;
  const bool fast = J.n_jobs <= 32 && J.n_mach <= 32 && J.per_job < 256 &&
                    J.n_jobs * J.per_job < 32768;
  for (int t = 0; t < m; ++t) {
    const int p = g.picks()[t];
    if (fast) {
      // the trials share the schedule up to the step where operation p becomes
      // a candidate: decode that prefix once per warp, then finish each trial
      const int jp = p / J.per_job, kp = p - jp * J.per_job;
      JspWarp base = jsp_warp_start(J, row, -1, 0, wl);
      jsp_warp_run(J, row, -1, 0, wl, base, jp, kp);
      // warp w takes trials [K w, K w + K) of each group of K * nwarps
      if (nd > 2 * nwarps) jsp_gr_trials<4>(J, row, g, base, jp, kp, nd, warp, nwarps, wl);
      else jsp_gr_trials<2>(J, row, g, base, jp, kp, nd, warp, nwarps, wl);
    } else {
      for (int i = warp; i < nd; i += nwarps) {
        const int sp = jsp_decode_warp(J, row, p, g.dom()[i], mf, wl);
        if (wl == 0) g.score()[i] = sp;
      }
    }
    team_bar(team, TS);
    if (lane == 0) {  // first minimum in domain order
      int bi = 0;
      for (int i = 1; i < nd; ++i)
        if (g.score()[i] < g.score()[bi]) bi = i;
      row[p] = (G)g.dom()[bi];
    }
    team_bar(team, TS);
  }
}

// Incremental trials for partitions.  A trial inserts v into one route r*;
// part_eval accumulates routes in order (Neumaier distance sum, capacity and
// lateness running sums), so the state after routes 0..r*-1 and the
// contributions of routes after r* are those of the row without v: cached
// once per value (thread 0, one pass in part_eval's order), then each trial
// only evaluates route r* and replays the cached terms.  Lateness terms that
// are 0.0 are not stored (adding +0.0 leaves a non-negative sum unchanged),
// so the result is bit-identical to part_eval_ins.
struct PartCache {
  double* rd;     // [d1] route distances
  double* over;   // [d1] capacity terms max(0, load - cap)
  double* ss;     // [d1] PySum state before route r
  double* sc;
  double* sf;
  double* cap;    // [d1] capacity sum before route r
  double* late;   // [d1] lateness sum before route r
  double* loff;   // [d1] start of route r's positive lateness terms in lt (cells before r + r)
  double* lcnt;   // [d1] how many
  double* lt;     // positive lateness terms, route r's at loff[r]
  __device__ __forceinline__ void bind(double* b, int d1) {
    rd = b;
    over = rd + d1;
    ss = over + d1;
    sc = ss + d1;
    sf = sc + d1;
    cap = sf + d1;
    late = cap + d1;
    loff = late + d1;
    lcnt = loff + d1;
    lt = lcnt + d1;
  }
  static __device__ __forceinline__ int doubles(int d1, int n) { return 9 * d1 + n + d1; }
};

// one route's (distance, capacity term, lateness terms) in part_eval's order
template <class R, class LT>
__device__ __forceinline__ void part_route(const PartView& v, const R& route, int len, double& rd,
                                           double& capterm, const LT& late_term) {
  const int n1 = v.n + 1;
  rd = 0.0;
  if (len > 0) {
    rd = __dadd_rn(v.dist[route[0] + 1], v.dist[(route[len - 1] + 1) * n1]);
    if (len > 1) {
      double acc = 0.0;
      if (len - 1 < 8) {  // np_pairwise small case, accessor inline
        acc = -0.0;
        for (int i = 0; i < len - 1; ++i)
          acc = __dadd_rn(acc, v.dist[(route[i] + 1) * n1 + route[i + 1] + 1]);
      } else {
        struct Edge {
          const double* d;
          const R* r;
          int n1;
          __device__ __forceinline__ double operator()(int i) const {
            return d[((*r)[i] + 1) * n1 + (*r)[i + 1] + 1];
          }
        } f{v.dist, &route, n1};
        acc = np_pairwise(f, 0, len - 1);
      }
      rd = __dadd_rn(rd, acc);
    }
  }
  struct Dem {
    const double* dem;
    const R* r;
    __device__ __forceinline__ double operator()(int i) const { return dem[(*r)[i]]; }
  } dm{v.demand, &route};
  const double load = np_pairwise(dm, 0, len);
  const double ov = __dsub_rn(load, v.cap);
  capterm = ov > 0.0 ? ov : 0.0;
  if (v.tw && len > 0) {
    double t = v.ready[0];
    int prev = 0;
    for (int q = 0; q < len; ++q) {
      const int node = route[q] + 1;
      const double arr0 = __dadd_rn(t, v.dist[prev * n1 + node]);
      const double arrival = v.ready[node] >= arr0 ? v.ready[node] : arr0;
      const double l = __dsub_rn(arrival, v.due[node]);
      if (l > 0.0) late_term(l);
      t = __dadd_rn(arrival, v.service[node]);
      prev = node;
    }
    const double back = __dsub_rn(__dadd_rn(t, v.dist[prev * n1]), v.due[0]);
    if (back > 0.0) late_term(back);
  }
}

struct PlainRoute {
  const short* b;
  __device__ __forceinline__ int operator[](int q) const { return b[q]; }
};

// routes in parallel (thread r: distance, capacity term, positive lateness
// terms), then thread 0 runs the prefix sums in part_eval's order
__device__ void part_cache_build(const PartView& v, const short* cells, const short* sz,
                                 PartCache& pc, int wl) {  // one warp
  for (int r = wl; r < v.d1; r += 32) {
    int at = 0;
    for (int q = 0; q < r; ++q) at += sz[q];
    const int base = at + r;
    int cnt = 0;
    double rd, ct;
    part_route(v, PlainRoute{cells + at}, sz[r], rd, ct, [&](double l) { pc.lt[base + cnt++] = l; });
    pc.rd[r] = rd;
    pc.over[r] = ct;
    pc.loff[r] = base;
    pc.lcnt[r] = cnt;
  }
  __syncwarp();
  if (wl == 0) {
    PySum ds;
    ds.init();
    double cap = 0.0, late = 0.0;
    for (int r = 0; r < v.d1; ++r) {
      pc.ss[r] = ds.s;
      pc.sc[r] = ds.c;
      pc.sf[r] = ds.first;
      pc.cap[r] = cap;
      pc.late[r] = late;
      ds.add(pc.rd[r]);
      cap = __dadd_rn(cap, pc.over[r]);
      const int b = (int)pc.loff[r], e = b + (int)pc.lcnt[r];
      for (int k = b; k < e; ++k) late = __dadd_rn(late, pc.lt[k]);
    }
  }
  __syncwarp();
}

// part_eval of the row with v inserted at (ri, pi), from the cache
__device__ __forceinline__ void part_eval_trial(const PartView& v, const short* cells,
                                                const short* sz, const PartCache& pc, int ri,
                                                int pi, int val, double& distance, double& penalty,
                                                int& veh) {
  PySum ds;
  ds.s = pc.ss[ri];
  ds.c = pc.sc[ri];
  ds.first = (int)pc.sf[ri];
  double cap = pc.cap[ri], late = pc.late[ri];
  int at = 0;
  veh = 0;
  for (int r = 0; r < v.d1; ++r) {
    if (r < ri) at += sz[r];
    veh += (sz[r] + (r == ri)) > 0;
  }
  double rd, ct;
  part_route(v, RouteIns{cells + at, pi, val}, sz[ri] + 1, rd, ct,
             [&](double l) { late = __dadd_rn(late, l); });
  ds.add(rd);
  cap = __dadd_rn(cap, ct);
  for (int r = ri + 1; r < v.d1; ++r) {
    ds.add(pc.rd[r]);
    cap = __dadd_rn(cap, pc.over[r]);
    const int b = (int)pc.loff[r], e = b + (int)pc.lcnt[r];
    for (int k = b; k < e; ++k) late = __dadd_rn(late, pc.lt[k]);
  }
  distance = ds.result();
  penalty = v.tw ? __dadd_rn(cap, late) : cap;
}

// scalar_fitness (engine.py:215-222) of a routing solution from its distance,
// penalty and vehicle count, objectives in the problem's order
__device__ __forceinline__ double part_scal(const RowArgs& X, double dist, int veh, double* o0,
                                            double* o1) {
  const double a = X.okind0 == 0 ? dist : (double)veh;
  const double b = X.okind1 == 0 ? dist : (double)veh;
  if (o0) *o0 = a;
  if (o1) *o1 = b;
  const double s = __dadd_rn(0.0, __dmul_rn(X.obj_weight, a));
  return X.mo.m == 2 ? __dadd_rn(s, __dmul_rn(X.w2, b)) : s;
}

// Φ of a partition candidate with the run's penalty weight (engine.py:215-222)
template <class U>
__device__ __forceinline__ double PartOpCtx<U>::phi() {
  double d, p;
  int veh;
  part_eval(pv, c->cells, c->sz, d, p, &veh);
  return __dadd_rn(part_scal(*X, d, veh, nullptr, nullptr), __dmul_rn(pw, p));
}

// Warp-cooperative edits of a compact partition row (cells, then the row sizes):
// the same removals / insertions as PartCtx::remove / insert, in the same order,
// with the O(n) shifts and the O(rows) scans spread over the 32 lanes.  Every
// lane returns the same value; the row is consistent after each call.
__device__ __forceinline__ int warp_row_start(const short* sz, int r, int wl) {
  int s = 0;
#pragma unroll 1
  for (int q = wl; q < r; q += 32) s += sz[q];
  return __reduce_add_sync(0xffffffffu, s);
}
__device__ __noinline__ short warp_cells_remove(short* cells, short* sz, int total, int r, int p,
                                                int wl) {
  const int gi = warp_row_start(sz, r, wl) + p;
  const short v = cells[gi];
#pragma unroll 1
  for (int base = gi; base < total - 1; base += 32) {  // ascending: a[q] = a[q + 1]
    const int q = base + wl;
    const short x = q < total - 1 ? cells[q + 1] : (short)0;
    __syncwarp();
    if (q < total - 1) cells[q] = x;
    __syncwarp();
  }
  if (wl == 0) sz[r] -= 1;
  __syncwarp();
  return v;
}
__device__ __noinline__ void warp_cells_insert(short* cells, short* sz, int total, int r, int p,
                                               short v, int wl) {
  const int gi = warp_row_start(sz, r, wl) + p;
#pragma unroll 1
  for (int top = total; top > gi; top -= 32) {  // descending: a[q] = a[q - 1]
    const int q = top - wl;
    const short x = q > gi ? cells[q - 1] : (short)0;
    __syncwarp();
    if (q > gi) cells[q] = x;
    __syncwarp();
  }
  if (wl == 0) {
    cells[gi] = v;
    sz[r] += 1;
  }
  __syncwarp();
}
// (row, position) of the cell holding value v
__device__ __noinline__ int2 warp_cells_find(const short* cells, const short* sz, int total, int d1,
                                             short v, int wl) {
  int gi = 0;
#pragma unroll 1
  for (int base = 0; base < total; base += 32) {
    const int q = base + wl;
    const unsigned hit = __ballot_sync(0xffffffffu, q < total && cells[q] == v);
    if (hit) {
      gi = base + __ffs(hit) - 1;
      break;
    }
  }
  // PartCtx::cell_at: first row whose running size exceeds gi
  int carry = 0;
#pragma unroll 1
  for (int base = 0; base < d1; base += 32) {
    const int q = base + wl;
    int incl = q < d1 ? sz[q] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (wl >= o) incl += y;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, q < d1 && gi < carry + incl);
    if (hit) {
      const int l = __ffs(hit) - 1;
      const int before = carry + __shfl_sync(0xffffffffu, incl, l) - sz[base + l];
      return make_int2(base + l, gi - before);
    }
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  return make_int2(d1 - 1, 0);
}

// partitions (operators.py:520-546): warp 0 pops / parks / re-inserts, the
// team scores every trial slot of every open row in parallel
__device__ void team_gr_part(const PartView& pv, short* cells, short* sz, int n_cells, int d1,
                             int d2, const RowArgs& X, double pw, const GrShared& g, double* sbuf,
                             TeamShared<double>* ts, int lane, int team, int TS) {
  const int m = g.m();
  if (m == 0) return;
  const int warp = lane >> 5, wl = lane & 31, nwarps = TS >> 5;
  if (warp == 0) {
    int total = n_cells;
    for (int t = 0; t < m; ++t) {
      const int rp = g.picks()[t];
      const short v = warp_cells_remove(cells, sz, total, rp >> 16, rp & 0xFFFF, wl);
      --total;
      if (wl == 0) g.taken()[t] = v;
    }
    for (int t = 0; t < m; ++t) {  // park at the end of the first open row
      int r = 0;
      while (r < d1 - 1 && sz[r] >= d2) ++r;
      warp_cells_insert(cells, sz, total, r, sz[r], (short)g.taken()[t], wl);
      ++total;
    }
  }
  // per pick: warp 0 alone re-inserts the previous value, pops this one and
  // builds the route cache; one team barrier, the trials, a second barrier
  PartCache pc;
  const bool cached = pv.variant == 0 && 32 + PartCache::doubles(d1, n_cells) <= 5 * TS;
  pc.bind(sbuf + 32, d1);
  for (int t = 0; t < m; ++t) {
    if (warp == 0) {
      const int2 rp = warp_cells_find(cells, sz, n_cells, d1, (short)g.taken()[t], wl);
      warp_cells_remove(cells, sz, n_cells, rp.x, rp.y, wl);
      if (cached) part_cache_build(pv, cells, sz, pc, wl);
    }
    team_bar(team, TS);  // the trials below read the row without v (and taken[], parked by warp 0)
    const short v = (short)g.taken()[t];
    int ntr = 0;  // trial slots: open rows in order, positions 0..sz[r]
    for (int r = 0; r < d1; ++r) ntr += sz[r] < d2 ? sz[r] + 1 : 0;
    double bs = 0.0;
    int bi = 0x7fffffff;
    for (int i = lane; i < ntr; i += TS) {
      int r = 0, k = i;
      for (; r < d1; ++r) {
        if (sz[r] >= d2) continue;
        if (k <= sz[r]) break;
        k -= sz[r] + 1;
      }
      double dist, pen;
      int veh;
      if (cached) part_eval_trial(pv, cells, sz, pc, r, k, v, dist, pen, veh);
      else {
        const PartEval e = part_eval_ins(pv, cells, sz, r, k, v);
        dist = e.distance;
        pen = e.penalty;
        veh = e.veh;
      }
      const double sc = __dadd_rn(part_scal(X, dist, veh, nullptr, nullptr), __dmul_rn(pw, pen));
      if (bi == 0x7fffffff || sc < bs) {
        bs = sc;
        bi = i;
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, bs, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (oi != 0x7fffffff && (bi == 0x7fffffff || ob < bs || (ob == bs && oi < bi))) {
        bs = ob;
        bi = oi;
      }
    }
    if (wl == 0) {
      sbuf[warp] = bs;
      ts->wl[warp] = bi;
    }
    team_bar(team, TS);
    if (warp == 0) {
      double b = 0.0;
      int ib = 0x7fffffff;
      for (int w = 0; w < nwarps; ++w) {
        const int oi = ts->wl[w];
        if (oi != 0x7fffffff && (ib == 0x7fffffff || sbuf[w] < b || (sbuf[w] == b && oi < ib))) {
          b = sbuf[w];
          ib = oi;
        }
      }
      int r = 0, k = ib;
      for (; r < d1; ++r) {
        if (sz[r] >= d2) continue;
        if (k <= sz[r]) break;
        k -= sz[r] + 1;
      }
      warp_cells_insert(cells, sz, n_cells - 1, r, k, v, wl);
    }
  }
  team_bar(team, TS);
}

// op_uniform_crossover (operators.py:451-462) resolved by one warp: lane 0 draws
// the mate (pick_mate may reject), then every cell's random() sits at a known
// word position (2 words each, no rejection), so the warp evaluates them in
// parallel from the counter-based stream.  Returns the stream position after
// the operator; lo/hi = touched range (hi <= lo: none).
template <class G>
__device__ __forceinline__ u32 warp_uniform_x(G* row, int n, const MateSel& ms, Stream& rng,
                                              int wl, int& lo, int& hi) {
  int mate = -1;
  u32 pos0 = 0;
  if (wl == 0) {
    const short* mp = ms.pick(rng);
    mate = mp ? (int)((mp - ms.rows) / n) : -1;
    pos0 = rng.tell();
  }
  mate = __shfl_sync(0xffffffffu, mate, 0);
  pos0 = __shfl_sync(0xffffffffu, pos0, 0);
  lo = n;
  hi = 0;
  if (mate < 0) return pos0;
  const short* mrow = ms.rows + (size_t)mate * n;
  // lane wl draws a contiguous run of cells, so consecutive random() calls
  // share Philox blocks (one block per two draws instead of one per draw); the
  // draws of a round of 32 cells become a bit mask, then the warp copies the
  // taken mate cells owner by owner with coalesced, independent loads (the
  // per-lane copy waited one L2 round trip per taken cell)
  const int c = (n + 31) >> 5, p0 = wl * c, p1 = p0 + c < n ? p0 + c : n;
  Stream r;
  r.k0 = rng.k0;
  r.k1 = rng.k1;
  if (p0 < p1) r.seek(pos0 + 2u * (u32)p0);
#pragma unroll 1
  for (int base = 0; base < c; base += 32) {
    unsigned mask = 0u;
#pragma unroll 1
    for (int i = 0; i < 32; ++i) {
      const int p = p0 + base + i;
      if (base + i >= c || p >= p1) break;
      if (r.random() < 0.5) mask |= 1u << i;
    }
    if (mask) {
      lo = min(lo, p0 + base + __ffs(mask) - 1);
      hi = p0 + base + 32 - __clz(mask);
    }
#pragma unroll 4
    for (int o = 0; o < 32; ++o) {  // owner lane o's cells p0(o) + base + wl
      const unsigned mo = __shfl_sync(0xffffffffu, mask, o);
      const int p = o * c + base + wl;
      if ((mo >> wl) & 1u) row[p] = (G)__ldcg(mrow + p);
    }
  }
  lo = (int)__reduce_min_sync(0xffffffffu, (unsigned)lo);
  hi = (int)__reduce_max_sync(0xffffffffu, (unsigned)hi);
  return pos0 + 2u * (u32)n;
}

// GO_ROW_TIMING (diagnostic build, tools/row_phase.py): team lane 0 charges
// clock64 intervals to prof[0..6] (copy, regroup, lane execution incl. the
// barrier wait, deferred uniform crossover, deferred guided rebuild, evaluation,
// acceptance), warp leaders their execution time to prof[8..11], and every lane
// the cycles of each operator kind to prof[12 + kind] (+ 2^40 per application).
#ifdef GO_ROW_TIMING
#define GO_RT_DECL unsigned long long rt_[8] = {0}, rt_last_ = clock64()
#define GO_RT(slot) do { const unsigned long long t_ = clock64(); rt_[(slot)] += t_ - rt_last_; rt_last_ = t_; } while (0)
#else
#define GO_RT_DECL do {} while (0)
#define GO_RT(slot) do {} while (0)
#endif

// RG: lane rows in global memory (long rows); a template constant so the
// shared-memory variant keeps ld.shared / st.shared on its lane rows
template <int KIND, class E, class G, class U = NoUser, bool RG = false>
__device__ __forceinline__ void evolve_row(const EvolveArgs& A, const RowArgs& X) {
  extern __shared__ __align__(128) unsigned char sm[];
  if (A.gs->stop) return;

  const unsigned ro = PermSmem::reg_off(A.inst_bytes);
  u64* mbar = (u64*)(sm + ro);
  double* s_cum = (double*)(sm + ro + 16);
  double* s_misc = s_cum + 32;
  int* s_kind = (int*)(s_misc + 4);
  int* s_gord = s_kind + 32;
  int* s_grank = s_gord + 32;
  const unsigned char* inst = (const unsigned char*)A.inst;
  int use_s = 0;
  if (A.inst_bytes) {
    stage_to_smem(sm, A.inst, A.inst_bytes, mbar);
    inst = sm;
    use_s = 1;
  }
  const RegistryDev* R = A.reg;
  const int nseq = R->nseq;
  for (int i = threadIdx.x; i < 32; i += blockDim.x) {
    s_cum[i] = R->cum[i];
    s_kind[i] = R->kind[i];
  }
  if (threadIdx.x < 3) s_misc[threadIdx.x] = R->kw[threadIdx.x];
  if (threadIdx.x == 3) s_misc[3] = R->total;
  if (threadIdx.x == blockDim.x - 1) {  // (a CTA may be a single 32-thread team)
    for (int i = 0; i < nseq; ++i) {
      s_gord[i] = i;
      s_grank[i] = i;
    }
  }
  __syncthreads();

  const int n = A.n;
  // problem views
  QapView<E> qv;
  KnapView kv;
  JspView jv;
  PartView pv;
  if (KIND == RK_PART) {
    pv.dist = (const double*)inst;
    pv.demand = (const double*)(inst + X.off1);
    pv.ready = (const double*)(inst + X.off2);
    pv.due = (const double*)(inst + X.off3);
    pv.service = (const double*)(inst + X.off4);
    pv.n = X.n_cells;
    pv.d1 = X.d1;
    pv.d2 = X.d2;
    pv.cap = X.capacity;
    pv.tw = X.tw;
    pv.variant = X.pvar;
    pv.prio = (const double*)(inst + X.off2);
  } else if (KIND == RK_QAP) {
    qv.f = (const E*)inst;
    qv.d = (const E*)(inst + X.off1);
    qv.n = n;
    qv.fs = use_s ? smem_u32(sm) : 0u;
    qv.ds = use_s ? smem_u32(sm + X.off1) : 0u;
    qv.use_s = use_s;
  } else if (KIND == RK_KNAP) {
    kv.w = (const double*)inst;
    kv.v = (const double*)(inst + X.off1);
    kv.cap = X.capacity;
  } else {
    jv.mach = (const int*)inst;
    jv.dur = (const int*)(inst + X.off1);
    jv.n_jobs = X.n_jobs;
    jv.per_job = X.per_job;
    jv.n_mach = X.n_mach;
  }

  const int TS = A.team_stride, T = A.T;
  const int team = threadIdx.x / TS, lane = threadIdx.x - team * TS;
  const int warp = lane >> 5, wl = lane & 31, nwarps = TS >> 5;
  const int ev = blockIdx.x * A.E + team;
  if (ev >= A.P) return;
  const long long evg = (long long)A.ev_offset + ev;

  const unsigned rs = RowSmem::row_stride(n, (int)sizeof(G));
  unsigned char* tb = sm + PermSmem::team_off(A.inst_bytes) + team * A.team_smem;
  G* cur = (G*)tb;
  // TS lane rows: shared memory after the current row, or (rows too long for
  // the opt-in shared memory) this team's slice of the global lane_rows buffer
  constexpr bool rows_g = RG;
  unsigned char* rows = rows_g ? (unsigned char*)A.lane_rows + (size_t)ev * TS * rs : tb + rs;
  unsigned char* lst = tb + RowSmem::align(rs * (rows_g ? 1 : TS + 1), 16);
  RowLaneState la;
  la.bind(lst, TS);
  TeamShared<double>* ts =
      (TeamShared<double>*)(lst + RowSmem::align(RowLaneState::bytes(TS), 16));
  int* scratch = (int*)((unsigned char*)ts + sizeof(TeamShared<double>));  // JSP decode

  for (int p = lane; p < n; p += TS) cur[p] = (G)A.genes[(size_t)ev * n + p];
  for (int i = lane; i < MAX_SEQ; i += TS) {
    ts->usage[i] = 0;
    ts->impr[i] = 0;
  }
  if (lane < 3) {
    ts->k_usage[lane] = 0;
    ts->k_impr[lane] = 0;
  }
  team_bar(team, TS);

  double scal = A.scal[ev], pen = A.pen[ev];
  double V = 0.0, W = 0.0;  // knapsack sums of the current row
  if (KIND == RK_KNAP || KIND == RK_QAP) {
    double pv = 0.0, pw = 0.0;
    if (KIND == RK_KNAP) {
      for (int p = lane; p < n; p += TS) {
        const double x = (double)cur[p];
        pv += kv.v[p] * x;
        pw += kv.w[p] * x;
      }
    } else {  // QAP: re-anchor Φ on an exact evaluation of the current row
      typedef typename AccOf<E>::T Aq;
      Aq s = 0;
      for (int i = lane; i < n; i += TS)
        for (int j = 0; j < n; ++j) s += qv.F(i, j) * qv.D(cur[i], cur[j]);
      pv = (double)s;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      pv += __shfl_xor_sync(0xffffffffu, pv, off);
      pw += __shfl_xor_sync(0xffffffffu, pw, off);
    }
    if (wl == 0) {
      ts->wd[warp] = pv;
      la.delta[warp] = pw;  // scratch use before the generation loop
    }
    team_bar(team, TS);
    double tv = 0.0, tw = 0.0;
    for (int w = 0; w < nwarps; ++w) {
      tv += ts->wd[w];
      tw += la.delta[w];
    }
    team_bar(team, TS);
    if (KIND == RK_KNAP) {
      V = tv;
      W = tw;
    } else {
      scal = tv;
    }
  }
  double bscal = A.best_scal[ev], bpen = A.best_pen[ev];
  // objective vectors of the current row and of the team best (multi-objective)
  double co0 = 0.0, co1 = 0.0, bo0 = 0.0, bo1 = 0.0;
  if (A.obj2) {
    co0 = A.obj2[2 * ev];
    co1 = A.obj2[2 * ev + 1];
    bo0 = A.best_obj2[2 * ev];
    bo1 = A.best_obj2[2 * ev + 1];
  }
  const double* kw = s_misc;
  const double total = s_misc[3];
  const unsigned lt_mask = (1u << wl) - 1u;
  int err = 0;
  unsigned long long rd_pos = 0, rd_elem = 0;
  const double pwt = X.penalty_weight;

  MateSel ms;
  int snap_min = (int)A.gen0;  // every team has published gen0 (host)
  GO_RT_DECL;
  for (int gi = 0; gi < A.ngen; ++gi) {
    const long long g = A.gen0 + gi;
    const double temp = A.temps[gi];
    GO_RT(6);
    // crossover snapshot of this generation (see EvolveArgs::snap)
    ms.init(A.snap, A.prog, (int)g, ev, A.P, A.islands, n);
#ifdef GO_PHASE_TIMING
    ms.prof = A.gs->prof;
#endif

    // ---- A: copy the current row into every lane row; draw k and sequence 0
    {
      const int words = (int)(rs / 16);
      const int4* src = (const int4*)cur;
      for (int idx = lane; idx < T * words; idx += TS) {
        const int L = idx / words, w = idx - L * words;
        ((int4*)(rows + (size_t)L * rs))[w] = src[w];
      }
    }
    if (lane < T) {
      Stream rng;
      rng.init(row_key_k<KIND>(A.seed, (u64)evg, (u64)g, (u64)lane, 0));
      const int k = sample_k(kw, rng);
      const int s0 = sample_seq(s_cum, nseq, total, rng);
      la.pos[lane] = rng.tell();
      la.meta[lane] = pack_meta(k, 0, s0, 0, 0);
      la.nr[lane] = 0;
    }
    team_bar(team, TS);

    GO_RT(0);
    // ---- B: chain steps, lanes regrouped by sequence ------------------------------
#pragma unroll 1
    for (int s = 0; s < MAX_CHAIN; ++s) {
      int hold_seq = 31;
      if (lane < T) {
        const u32 mt = la.meta[lane];
        if (meta_k(mt) > s) hold_seq = meta_sq(mt, s);
      }
      const unsigned grp = __match_any_sync(0xffffffffu, hold_seq);
      const int rank = __popc(grp & lt_mask);
      ts->cnt[warp][wl] = 0;
      __syncwarp();
      if (hold_seq != 31 && rank == 0) ts->cnt[warp][hold_seq] = (unsigned char)__popc(grp);
      team_bar(team, TS);
      if (lane == 0) {  // after the barrier: every thread has read the previous step's counts
        ts->nreq = 0;
        ts->ndreq = 0;
        ts->ngr = 0;
      }
      int tj = 0;
      if (wl < nseq) {
        const int q = s_gord[wl];
        for (int w = 0; w < nwarps; ++w) tj += ts->cnt[w][q];
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
        for (int w = 0; w < warp; ++w) base += ts->cnt[w][hold_seq];
        la.order[base + rank] = (unsigned short)lane;
      }
      team_bar(team, TS);
      GO_RT(1);
#ifdef GO_ROW_TIMING
      const unsigned long long t_ex0 = clock64();
#endif
      if (active == 0) break;

      // Two passes over the lanes' operators.  Pass 0 runs this step's lanes but
      // defers OX crossovers, which may wait for a mate team's snapshot of this
      // generation; pass 1 runs them after the team's guided rebuilds and the
      // uniform crossovers (warp-resolved, also mate-bound), so the wait
      // overlaps work that needs no mate.  Lanes are independent and each keeps
      // its own stream position, so the order between lanes changes no result.
      // (ts->ngr counts the deferred OX lanes, queued from the back of uxreq.)
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        const int nitems = pass == 0 ? active : ts->ngr;
        if (pass == 1 && nitems == 0) break;
        // item i runs on warp (i / 32 + team) mod nwarps: a CTA's warp w runs
        // on scheduler w mod 4, so the teams' equal sort orders would otherwise
        // put every team's most expensive sequence groups on one scheduler
        const int item = ((warp + nwarps - team % nwarps) % nwarps) * 32 + wl;
        if (item < nitems) {
          const int L = pass == 0 ? la.order[item] : la.uxreq[TS - 1 - item];
          Stream rng;
          rng.init(row_key_k<KIND>(A.seed, (u64)evg, (u64)g, (u64)L, 0));
          rng.seek(la.pos[L]);
          const u32 meta = la.meta[L];
          const int k = meta_k(meta);
          int q0 = meta_sq(meta, 0), q1 = meta_sq(meta, 1), q2 = meta_sq(meta, 2);
          bool pending = false;
          if constexpr (KIND == RK_PART) {
            PartCtx c;
            c.rng = rng;
            c.cells = (short*)(rows + (size_t)L * rs);
            c.sz = c.cells + X.n_cells;
            c.n = X.n_cells;
            c.d1 = X.d1;
            c.d2 = X.d2;
            c.n_cfg = X.n_cfg;
            c.total = X.n_cells;
            c.err = 0;
            c.mates = &ms;
            const int kind = s_kind[s == 0 ? q0 : (s == 1 ? q1 : q2)];
            if (kind == SEQ_GUIDED_REBUILD) {  // team-resolved below
              la.greq[atomicAdd(&ts->nreq, 1)] = (unsigned short)L;
              pending = true;
            } else if (pass == 0 && kind == SEQ_OX) {  // after the rebuilds (pass 1)
              la.uxreq[TS - 1 - atomicAdd(&ts->ngr, 1)] = (unsigned short)L;
              pending = true;
            } else if (U::kHasOps && kind >= SEQ_CUSTOM_BASE) {  // user operator (register_custom)
              if constexpr (U::kHasOps) {
                PartOpCtx<U> oc{&c, pv, &X, pwt, X.n_cells, X.d1, X.d2};
                U::op(kind - SEQ_CUSTOM_BASE, oc, inst);
              }
            } else {
              {
  #ifdef GO_ROW_TIMING
                const unsigned long long t_op = clock64();
  #endif
                run_part_op(kind, c);
  #ifdef GO_ROW_TIMING
                if (kind < 16) atomicAdd(&A.gs->prof[12 + kind], (clock64() - t_op) + (1ull << 40));
  #endif
              }
            }
            rng = c.rng;
            err |= c.err;
          } else {
            RowCtx<G> c;
            c.rng = rng;
            c.row = (G*)(rows + (size_t)L * rs);
            c.full = c.row;
            c.mf = X.mf;
            c.d1 = X.mf ? X.d1 : 1;
            c.d2 = X.d2;
            c.n = X.mf == 1 ? X.d2 : n;  // permutation rows: ops see one row
            c.n_cfg = X.n_cfg;
            c.lb = X.lb;
            c.ub = X.ub;
            c.err = 0;
            c.nr = la.nr[L];
            c.rlo = la.rlo + L;
            c.rhi = la.rhi + L;
            c.rstride = TS;
            c.mates = &ms;
            const int kind = s_kind[s == 0 ? q0 : (s == 1 ? q1 : q2)];
            if (kind == SEQ_GUIDED_REBUILD && KIND == RK_KNAP) {  // O(1) trials: inline
              gr_cells<KIND>(kv, jv, c.row, n, X.n_cfg, X.lb, X.ub, X.obj_weight, pwt,
                             scratch + L * X.scratch_ints, c);
              c.mark_all();
            } else if (kind == SEQ_GUIDED_REBUILD) {  // team-resolved below
              la.greq[atomicAdd(&ts->nreq, 1)] = (unsigned short)L;
              pending = true;
            } else if (kind == SEQ_UNIFORM_X) {  // warp-resolved below
              la.uxreq[atomicAdd(&ts->ndreq, 1)] = (unsigned short)L;
              pending = true;
            } else if (pass == 0 && kind == SEQ_OX) {  // after the rebuilds (pass 1)
              la.uxreq[TS - 1 - atomicAdd(&ts->ngr, 1)] = (unsigned short)L;
              pending = true;
            } else if (U::kHasOps && kind >= SEQ_CUSTOM_BASE) {  // user operator (register_custom)
              if constexpr (U::kHasOps) {
              RowInst ri{inst, X.off1, KIND == RK_QAP ? RI_QAP : (KIND == RK_KNAP ? RI_KNAP :
                                                                   (KIND == RK_JSP ? RI_JSP : RI_NONE)),
                         KIND == RK_QAP ? (int)sizeof(E) : 8, n, X.capacity, n};
              RowOpCtx<G, U> oc{&c, UserScore{inst, X.obj_weight, pwt, X.mo.maxmask, X.w2, X.mo.m},
                                n, c.d1, X.d2, ri};
              U::op(kind - SEQ_CUSTOM_BASE, oc, inst);
              c.mark_all();
              }
            } else {
              {
  #ifdef GO_ROW_TIMING
                const unsigned long long t_op = clock64();
  #endif
                run_row_op(kind, c);
  #ifdef GO_ROW_TIMING
                if (kind < 16) atomicAdd(&A.gs->prof[12 + kind], (clock64() - t_op) + (1ull << 40));
  #endif
              }
            }
            rng = c.rng;
            err |= c.err;
            la.nr[L] = (unsigned char)(c.nr > MAX_RANGES ? MAX_RANGES + 1 : c.nr);
          }
          if (!pending) {
            if (s + 1 < k) {
              const int nq = sample_seq(s_cum, nseq, total, rng);
              if (s == 0) q1 = nq; else q2 = nq;
            }
            la.pos[L] = rng.tell();
            la.meta[L] = pack_meta(k, 0, q0, q1, q2);
          }
        }
#ifdef GO_ROW_TIMING
        if (pass == 0 && wl == 0 && warp < 4) atomicAdd(&A.gs->prof[8 + warp], clock64() - t_ex0);
#endif
        team_bar(team, TS);
        GO_RT(2);
        if (pass == 1) break;

        // ---- deferred guided rebuilds: the whole team, one lane at a time ------------
        const int ngr = ts->nreq;
        if (ngr > 0) {
          const GrShared gsh{(int*)&ts->cnt[0][0]};
  #pragma unroll 1
          for (int r = 0; r < ngr; ++r) {
            const int L = la.greq[r];
            G* lrow = (G*)(rows + (size_t)L * rs);
            if (lane == 0) {
              Stream rng;
              rng.init(row_key_k<KIND>(A.seed, (u64)evg, (u64)g, (u64)L, 0));
              rng.seek(la.pos[L]);
              // MULTI_FIXED permutation rows: home_row = randrange(d1) (operators.py:519-521)
              gsh.row() = (KIND == RK_USER && X.mf == 1) ? rng.randbelow(X.d1) : 0;
              gr_draw<KIND>(rng, gsh, KIND == RK_PART ? X.n_cells : (X.mf == 1 ? X.d2 : n), X.n_cfg,
                            X.lb, X.ub,
                            (const short*)lrow + X.n_cells, X.d1,
                            KIND == RK_JSP || (KIND == RK_USER && X.enc != ENC_PERM));
              const u32 meta = la.meta[L];
              const int k = meta_k(meta);
              int q1 = meta_sq(meta, 1), q2 = meta_sq(meta, 2);
              if (s + 1 < k) {
                const int nq = sample_seq(s_cum, nseq, total, rng);
                if (s == 0) q1 = nq; else q2 = nq;
              }
              la.pos[L] = rng.tell();
              la.meta[L] = pack_meta(k, 0, meta_sq(meta, 0), q1, q2);
              la.nr[L] = (unsigned char)(MAX_RANGES + 1);  // whole row re-evaluated
            }
            team_bar(team, TS);
            if (KIND == RK_QAP) {
              team_gr_qap(qv, lrow, n, gsh, la.delta, lane, team, TS);
            } else if (KIND == RK_JSP) {
              team_gr_jsp(jv, lrow, gsh, scratch, X.scratch_ints, lane, team, TS);
            } else if (KIND == RK_PART) {
              team_gr_part(pv, (short*)lrow, (short*)lrow + X.n_cells, X.n_cells, X.d1, X.d2, X,
                           pwt, gsh, la.delta, ts, lane, team, TS);
            } else if (KIND == RK_USER) {
              const UserScore us{inst, X.obj_weight, pwt, X.mo.maxmask, X.w2, X.mo.m};
              if (X.enc == ENC_PERM)
                team_gr_user_perm<U>(lrow, n, gsh.row() * X.d2, X.mf == 1 ? X.d2 : n, gsh, us,
                                     la.delta, ts, lane, team, TS);
              else
                team_gr_user_cells<U>(lrow, n, gsh, us, la.delta, lane, team, TS);
            }
            team_bar(team, TS);
          }
        }
        GO_RT(4);
        // ---- deferred uniform crossovers: one warp per lane -------------------------
        const int nux = ts->ndreq;
        if (nux > 0) {
  #pragma unroll 1
          for (int r = warp; r < nux; r += nwarps) {
            const int L = la.uxreq[r];
            Stream rng;
            rng.init(row_key_k<KIND>(A.seed, (u64)evg, (u64)g, (u64)L, 0));
            rng.seek(la.pos[L]);
            int lo, hi;
            const u32 pend = warp_uniform_x((G*)(rows + (size_t)L * rs), n, ms, rng, wl, lo, hi);
            __syncwarp();  // every lane has read la.pos before lane 0 updates it
            if (wl == 0) {
              rng.seek(pend);
              const u32 meta = la.meta[L];
              const int k = meta_k(meta);
              int q1 = meta_sq(meta, 1), q2 = meta_sq(meta, 2);
              if (s + 1 < k) {
                const int nq = sample_seq(s_cum, nseq, total, rng);
                if (s == 0) q1 = nq; else q2 = nq;
              }
              la.pos[L] = rng.tell();
              la.meta[L] = pack_meta(k, 0, meta_sq(meta, 0), q1, q2);
              if (hi > lo) {  // RowCtx::mark
                const int nr = la.nr[L];
                if (nr < MAX_RANGES) {
                  la.rlo[nr * TS + L] = (short)lo;
                  la.rhi[nr * TS + L] = (short)hi;
                }
                la.nr[L] = (unsigned char)(nr + 1 > MAX_RANGES ? MAX_RANGES + 1 : nr + 1);
              }
            }
          }
          team_bar(team, TS);
        }

        GO_RT(3);
      }
    }

    GO_RT(4);
    // ---- C: evaluate every lane (identity mapping) --------------------------------
    constexpr bool kQapInt = KIND == RK_QAP && AccOf<E>::kInt;
    if constexpr (kQapInt) {  // team-cooperative deltas (team_qap_delta_int)
      int t = 0;
      if (lane < T) {
        const int nr = la.nr[lane];
        int lo[MAX_RANGES], hi[MAX_RANGES];
        short l_in[MAX_RANGES], h_in[MAX_RANGES];
        for (int r = 0; r < nr && r < MAX_RANGES; ++r) {
          l_in[r] = la.rlo[r * TS + lane];
          h_in[r] = la.rhi[r * TS + lane];
        }
        const int nm = merge_ranges(nr, l_in, h_in, n, lo, hi);
        if (nm < 0) {
          t = n;
          la.nr[lane] = 255;
        } else {
          la.nr[lane] = (unsigned char)nm;
#pragma unroll 1
          for (int r = 0; r < nm; ++r) {
            la.rlo[r * TS + lane] = (short)lo[r];
            la.rhi[r * TS + lane] = (short)hi[r];
            t += hi[r] - lo[r];
          }
        }
        rd_elem += nm < 0 ? 3u * (unsigned)(n * n) : 3u * (unsigned)(n * t);
        rd_pos += 2u * (unsigned)n;
      }
      ((unsigned long long*)la.delta)[lane] = 0ull;
      ((int*)la.nscal)[lane] = t;
      if (qv.use_s) team_qap_delta_int<true>(qv, cur, rows, rs, la, ts->wl, lane, team, TS);
      else team_qap_delta_int<false>(qv, cur, rows, rs, la, ts->wl, lane, team, TS);
      team_bar(team, TS);
      if (lane < T) {
        const double dq = (double)(long long)((unsigned long long*)la.delta)[lane];
        la.delta[lane] = dq;
        la.nscal[lane] = scal + dq;
        la.npen[lane] = pen;
        la.aux0[lane] = 0.0;
        la.aux1[lane] = 0.0;
      }
    }
    if (!kQapInt && lane < T) {
      const G* row = (const G*)(rows + (size_t)lane * rs);
      int lo[MAX_RANGES], hi[MAX_RANGES];
      short l_in[MAX_RANGES], h_in[MAX_RANGES];
      const int nr = la.nr[lane];
      for (int r = 0; r < nr && r < MAX_RANGES; ++r) {
        l_in[r] = la.rlo[r * TS + lane];
        h_in[r] = la.rhi[r * TS + lane];
      }
      const int nm = merge_ranges(nr, l_in, h_in, n, lo, hi);
      double nscal = scal, npen = pen, a0 = 0.0, a1 = 0.0, dl;
      if (KIND == RK_PART) {
        double dist, pn;
        int veh;
        part_eval(pv, (const short*)row, (const short*)row + X.n_cells, dist, pn, &veh);
        nscal = part_scal(X, dist, veh, &a0, &a1);  // a0 / a1: objective vector
        npen = pn;
        if (X.mo.lex) {
          dl = lex_delta(a0, a1, npen, co0, co1, pen, pwt, X.mo);
        } else {
          const double phi_c = __dadd_rn(nscal, __dmul_rn(pwt, npen));
          const double phi0 = __dadd_rn(scal, __dmul_rn(pwt, pen));
          dl = __dsub_rn(phi_c, phi0);
        }
        rd_elem += 6u * (unsigned)X.n_cells;
      } else if (KIND == RK_USER) {  // NVRTC objective(s), full evaluation
        const RowSol<G> sol{row, n};
        a0 = U::obj(sol, inst);
        nscal = __dadd_rn(0.0, __dmul_rn(X.obj_weight, (X.mo.maxmask & 1) ? -a0 : a0));
        if (X.mo.m == 2) {
          a1 = U::obj2(sol, inst);
          nscal = __dadd_rn(nscal, __dmul_rn(X.w2, (X.mo.maxmask & 2) ? -a1 : a1));
        }
        npen = U::pen(sol, inst);
        if (X.mo.lex) {
          dl = lex_delta(a0, a1, npen, co0, co1, pen, pwt, X.mo);
        } else {
          const double phi_c = __dadd_rn(nscal, __dmul_rn(pwt, npen));
          const double phi0 = __dadd_rn(scal, __dmul_rn(pwt, pen));
          dl = __dsub_rn(phi_c, phi0);
        }
      } else if (KIND == RK_QAP) {
        unsigned rd = 0;
        const double dq = qap_delta(qv, cur, row, nm, lo, hi, rd);
        rd_elem += rd;
        nscal = scal + dq;
        dl = dq;
      } else if (KIND == RK_KNAP) {
        double dv, dw;
        knap_delta(kv, cur, row, n, nm, lo, hi, dv, dw);
        const double nv = V + dv, nw = W + dw;
        const double over = __dsub_rn(nw, kv.cap);
        npen = over > 0.0 ? over : 0.0;
        nscal = __dadd_rn(0.0, __dmul_rn(X.obj_weight, -nv));
        const double phi_c = __dadd_rn(nscal, __dmul_rn(pwt, npen));
        const double phi0 = __dadd_rn(scal, __dmul_rn(pwt, pen));
        dl = __dsub_rn(phi_c, phi0);
        a0 = nv;
        a1 = nw;
        rd_elem += 2u * (unsigned)n;
      } else {
        const int span = jsp_decode(jv, row, scratch + lane * X.scratch_ints);
        nscal = (double)span;
        dl = nscal - scal;
        rd_elem += (unsigned)(n * jv.n_jobs);
      }
      la.delta[lane] = dl;
      la.nscal[lane] = nscal;
      la.npen[lane] = npen;
      la.aux0[lane] = a0;
      la.aux1[lane] = a1;
      rd_pos += 2u * (unsigned)n;
    }

    GO_RT(5);
    // ---- argmin over (delta, lane), acceptance, credit ----------------------------
    double bd = lane < T ? la.delta[lane] : 1.7976931348623157e308;
    int bl = lane < T ? lane : 0x7fffffff;
    argmin_warp(bd, bl);
    if (wl == 0) {
      ts->wd[warp] = bd;
      ts->wl[warp] = bl;
    }
    team_bar(team, TS);
    bd = ts->wd[0];
    bl = ts->wl[0];
    for (int w = 1; w < nwarps; ++w) {
      const double od = ts->wd[w];
      if (od < bd) {
        bd = od;
        bl = ts->wl[w];
      }
    }
    if (lane == 0) {
      int acc = bd < 0.0;
      if (!acc && temp > 0.0) {
        Stream ar;
        ar.init(row_key_k<KIND>(A.seed, (u64)evg, (u64)g, 0, 1));
        acc = ar.random() < exp(-bd / temp);
      }
      ts->accept = acc;
      if (acc) {
        const u32 meta = la.meta[bl];
        const int kk = meta_k(meta);
        const int improved = bd < 0.0;
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
      const int4* src = (const int4*)(rows + (size_t)bl * rs);
      for (int w = lane; w < (int)(rs / 16); w += TS) ((int4*)cur)[w] = src[w];
      scal = la.nscal[bl];
      pen = la.npen[bl];
      V = la.aux0[bl];
      W = la.aux1[bl];
      co0 = la.aux0[bl];  // routing: objective vector of the winner
      co1 = la.aux1[bl];
      team_bar(team, TS);
    }
    if (A.rec_obj2 && lane == 0) {
      A.rec_obj2[((size_t)gi * A.P + ev) * 2] = co0;
      A.rec_obj2[((size_t)gi * A.P + ev) * 2 + 1] = co1;
    }
    if (lane == 0) {
      A.rec_scal[(size_t)gi * A.P + ev] = scal;
      A.rec_pen[(size_t)gi * A.P + ev] = pen;
    }
    if (A.snap && gi + 1 < A.ngen)
      snap_publish(A.snap, A.prog, A.P, ev, n, (int)g + 1, cur, snap_min, lane, team, TS);
    if (compare_mo(pen, scal, co0, co1, bpen, bscal, bo0, bo1, X.mo) < 0 && !target_reached(A, bpen, bscal)) {
      for (int p = lane; p < n; p += TS) A.best_genes[(size_t)ev * n + p] = (short)cur[p];
      bscal = scal;
      bpen = pen;
      bo0 = co0;
      bo1 = co1;
      if (lane == 0) A.best_gen[ev] = g;
    }
  }

  team_bar(team, TS);
  for (int p = lane; p < n; p += TS) A.genes[(size_t)ev * n + p] = (short)cur[p];
  for (int i = lane; i < MAX_SEQ; i += TS) {
    A.usage[ev * MAX_SEQ + i] = ts->usage[i];
    A.impr[ev * MAX_SEQ + i] = ts->impr[i];
  }
  if (lane < 3) {
    A.k_usage[ev * 3 + lane] = ts->k_usage[lane];
    A.k_impr[ev * 3 + lane] = ts->k_impr[lane];
  }
  if (lane == 0) {
    A.scal[ev] = scal;
    A.pen[ev] = pen;
    A.best_scal[ev] = bscal;
    A.best_pen[ev] = bpen;
    if (A.obj2) {
      A.obj2[2 * ev] = co0;
      A.obj2[2 * ev + 1] = co1;
      A.best_obj2[2 * ev] = bo0;
      A.best_obj2[2 * ev + 1] = bo1;
    }
  }
#ifdef GO_ROW_TIMING
  if (lane == 0)
    for (int i = 0; i < 7; ++i) atomicAdd(&A.gs->prof[i], rt_[i]);
#endif
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
