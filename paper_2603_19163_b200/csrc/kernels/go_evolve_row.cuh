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

enum RowKind { RK_QAP = 0, RK_KNAP = 1, RK_JSP = 2, RK_PART = 3 };

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
  static __host__ __device__ unsigned bytes(int TS) {
    return (unsigned)(TS * (4 + 4 + 8 * 5 + 2 + 1 + 4 * MAX_RANGES) + 16);
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
  }
};

struct RowSmem {
  static __host__ __device__ unsigned align(unsigned x, unsigned a) { return (x + a - 1) / a * a; }
  static __host__ __device__ unsigned row_stride(int n, int gsize) { return align((unsigned)(n * gsize), 16); }
  static __host__ __device__ unsigned team_bytes(int n, int gsize, int TS, int scratch_per_lane) {
    return align(row_stride(n, gsize) * (TS + 1) + RowLaneState::bytes(TS) +
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
  // pairs with i touched
  for (int r = 0; r < nm; ++r)
    for (int i = lo[r]; i < hi[r]; ++i) {
      const int pi = row[i], ci = cur[i];
      for (int j = 0; j < n; ++j) d += q.F(i, j) * (q.D(pi, row[j]) - q.D(ci, cur[j]));
      rd += 3u * (unsigned)n;
    }
  // pairs with only j touched
  int gap_lo = 0;
  for (int r = 0; r <= nm; ++r) {
    const int gap_hi = r < nm ? lo[r] : n;
    for (int i = gap_lo; i < gap_hi; ++i) {
      const int ci = cur[i];
      for (int s = 0; s < nm; ++s)
        for (int j = lo[s]; j < hi[s]; ++j) d += q.F(i, j) * (q.D(ci, row[j]) - q.D(ci, cur[j]));
    }
    if (r < nm) gap_lo = hi[r];
  }
  return (double)d;
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
__host__ __device__ __forceinline__ int jsp_scratch_ints(int n_jobs, int n_mach) {
  return n_jobs + n_mach + (n_jobs + 3) / 4;
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

template <class E, class G, class R>
__device__ void gr_qap(const QapView<E>& q, G* row, int n, int n_cfg, R& rng) {
  typedef typename AccOf<E>::T A;
  if (n < 3) return;
  const int ls = lns_scope(n_cfg);
  const int m = ls < n - 1 ? ls : n - 1;
  int picks[30];
  G taken[30];
  sample_range(rng, n, m, picks);
  sort_desc(picks, m);
  int size = n;
  for (int t = 0; t < m; ++t) {  // _row_remove in (r, -p) order
    taken[t] = row[picks[t]];
    row_pop(row, size, picks[t]);
    --size;
  }
  for (int t = 0; t < m; ++t) row[size++] = taken[t];  // park at the row end
  for (int t = 0; t < m; ++t) {
    const G v = taken[t];
    int q0 = 0;
    while (row[q0] != v) ++q0;
    row_pop(row, n, q0);
    row[n - 1] = v;  // trial n-1 (score offset 0), then walk down to 0
    A sc = 0, best = 0;
    int bp = n - 1;
    for (int p = n - 1; p >= 1; --p) {
      sc += qap_swap_delta(q, row, n, p - 1, p);
      const G tmp = row[p - 1];
      row[p - 1] = row[p];
      row[p] = tmp;
      if (sc <= best) {  // lower positions win ties: first minimum in 0..n-1
        best = sc;
        bp = p - 1;
      }
    }
    for (int p = 0; p < bp; ++p) row[p] = row[p + 1];  // v from 0 to bp
    row[bp] = v;
  }
}

// binary / integer: coordinate-greedy reset of a scatter of cells
template <int KIND, class G, class R>
__device__ void gr_cells(const KnapView& kv, const JspView& jv, G* row, int n, int n_cfg, int lb,
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

// partitions (VRPTW / CVRP): operators.py:520-546 with a full evaluation per trial
__device__ void gr_part(const PartView& pv, PartCtx& c, double wobj, double pw) {
  const int total = c.total;
  if (total < 3) return;
  const int ls = lns_scope(c.n_cfg);
  const int m = ls < total - 1 ? ls : total - 1;
  int picks[30], rr[30], pp[30];
  short taken[30];
  sample_range(c, total, m, picks);
  for (int t = 0; t < m; ++t) c.cell_at(picks[t], rr[t], pp[t]);
  for (int i = 1; i < m; ++i) {  // sorted by (r, -p)
    const int r0 = rr[i], p0 = pp[i];
    int j = i;
    while (j > 0 && (rr[j - 1] > r0 || (rr[j - 1] == r0 && pp[j - 1] < p0))) {
      rr[j] = rr[j - 1];
      pp[j] = pp[j - 1];
      --j;
    }
    rr[j] = r0;
    pp[j] = p0;
  }
  for (int t = 0; t < m; ++t) taken[t] = c.remove(rr[t], pp[t]);
  for (int t = 0; t < m; ++t) {  // park at the end of the first open row
    int r = 0;
    while (r < c.d1 - 1 && c.sz[r] >= c.d2) ++r;
    c.insert(r, c.sz[r], taken[t]);
  }
  for (int t = 0; t < m; ++t) {
    const short v = taken[t];
    int g = 0;
    while (c.cells[g] != v) ++g;
    int r0, p0;
    c.cell_at(g, r0, p0);
    c.remove(r0, p0);
    double bs = 0.0;
    int br = -1, bp = 0;
    for (int r = 0; r < c.d1; ++r) {
      if (c.sz[r] >= c.d2) continue;
      const int lim = c.sz[r];
      for (int pos = 0; pos <= lim; ++pos) {
        c.insert(r, pos, v);
        double dist, pen;
        part_eval(pv, c.cells, c.sz, dist, pen);
        const double sc = __dadd_rn(__dadd_rn(0.0, __dmul_rn(wobj, dist)), __dmul_rn(pw, pen));
        c.remove(r, pos);
        if (br < 0 || sc < bs) {
          bs = sc;
          br = r;
          bp = pos;
        }
      }
    }
    c.insert(br, bp, v);
  }
}

template <int KIND, class E, class G>
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
  if (threadIdx.x == 32) {
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
  unsigned char* rows = tb + rs;  // TS lane rows
  RowLaneState la;
  la.bind(tb + rs * (TS + 1), TS);
  TeamShared<double>* ts =
      (TeamShared<double>*)(tb + rs * (TS + 1) + RowSmem::align(RowLaneState::bytes(TS), 16));
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
  const double* kw = s_misc;
  const double total = s_misc[3];
  const unsigned lt_mask = (1u << wl) - 1u;
  int err = 0;
  unsigned long long rd_pos = 0, rd_elem = 0;
  const double pwt = X.penalty_weight;

  MateSel ms;
  for (int gi = 0; gi < A.ngen; ++gi) {
    const long long g = A.gen0 + gi;
    const double temp = A.temps[gi];
    // crossover snapshot of this generation (see EvolveArgs::snap)
    if (A.snap && gi > 0) grid_team_barrier(A.gbar, (unsigned)(gi * A.P), lane, team, TS);
    ms.init(A.snap ? A.snap + (size_t)(g & 1) * A.P * n : nullptr, ev, A.P, A.islands, n);

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
      rng.init(mix64_5(A.seed, (u64)evg, (u64)g, (u64)lane, 0));
      const int k = sample_k(kw, rng);
      const int s0 = sample_seq(s_cum, nseq, total, rng);
      la.pos[lane] = rng.tell();
      la.meta[lane] = pack_meta(k, 0, s0, 0, 0);
      la.nr[lane] = 0;
    }
    team_bar(team, TS);

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
      if (active == 0) break;

      if (lane < active) {
        const int L = la.order[lane];
        Stream rng;
        rng.init(mix64_5(A.seed, (u64)evg, (u64)g, (u64)L, 0));
        rng.seek(la.pos[L]);
        const u32 meta = la.meta[L];
        const int k = meta_k(meta);
        int q0 = meta_sq(meta, 0), q1 = meta_sq(meta, 1), q2 = meta_sq(meta, 2);
        if (KIND == RK_PART) {
          PartCtx c;
          c.rng = &rng;
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
          if (kind == SEQ_GUIDED_REBUILD) gr_part(pv, c, X.obj_weight, pwt);
          else run_part_op(kind, c);
          err |= c.err;
        } else {
          RowCtx<G> c;
          c.rng = &rng;
          c.row = (G*)(rows + (size_t)L * rs);
          c.n = n;
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
          if (kind == SEQ_GUIDED_REBUILD) {
            if (KIND == RK_QAP) gr_qap(qv, c.row, n, X.n_cfg, c);
            else gr_cells<KIND>(kv, jv, c.row, n, X.n_cfg, X.lb, X.ub, X.obj_weight, pwt,
                                scratch + L * X.scratch_ints, c);
            c.mark_all();
          } else {
            run_row_op(kind, c);
          }
          err |= c.err;
          la.nr[L] = (unsigned char)(c.nr > MAX_RANGES ? MAX_RANGES + 1 : c.nr);
        }
        if (s + 1 < k) {
          const int nq = sample_seq(s_cum, nseq, total, rng);
          if (s == 0) q1 = nq; else q2 = nq;
        }
        la.pos[L] = rng.tell();
        la.meta[L] = pack_meta(k, 0, q0, q1, q2);
      }
      team_bar(team, TS);
    }

    // ---- C: evaluate every lane (identity mapping) --------------------------------
    if (lane < T) {
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
        part_eval(pv, (const short*)row, (const short*)row + X.n_cells, dist, pn);
        nscal = __dadd_rn(0.0, __dmul_rn(X.obj_weight, dist));
        npen = pn;
        const double phi_c = __dadd_rn(nscal, __dmul_rn(pwt, npen));
        const double phi0 = __dadd_rn(scal, __dmul_rn(pwt, pen));
        dl = __dsub_rn(phi_c, phi0);
        rd_elem += 6u * (unsigned)X.n_cells;
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
        ar.init(mix64_5(A.seed, (u64)evg, (u64)g, 0, 1));
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
      team_bar(team, TS);
    }
    if (lane == 0) {
      A.rec_scal[(size_t)gi * A.P + ev] = scal;
      A.rec_pen[(size_t)gi * A.P + ev] = pen;
    }
    if (A.snap && gi + 1 < A.ngen) {
      short* sn = A.snap + ((size_t)((g + 1) & 1) * A.P + ev) * n;
      for (int p = lane; p < n; p += TS) sn[p] = (short)cur[p];
    }
    if (strictly_better(pen, scal, bpen, bscal)) {
      for (int p = lane; p < n; p += TS) A.best_genes[(size_t)ev * n + p] = (short)cur[p];
      bscal = scal;
      bpen = pen;
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
