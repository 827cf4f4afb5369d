// go_row_entry.cuh — kernels of the row family (QAP / knapsack / JSP-int).
#pragma once
#include "go_evolve_row.cuh"

namespace go {

// evaluate() for m QAP permutations (builtins.py:282-284), one block each
template <class E>
__device__ __forceinline__ void qap_eval_entry(const void* inst, unsigned off1, int n,
                                               const short* genes, double* obj) {
  typedef typename AccOf<E>::T A;
  __shared__ A red[32];
  const E* f = (const E*)inst;
  const E* d = (const E*)((const unsigned char*)inst + off1);
  const short* p = genes + (size_t)blockIdx.x * n;
  A s = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    for (int j = 0; j < n; ++j) s += (A)f[i * n + j] * (A)d[p[i] * n + p[j]];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    A t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    obj[blockIdx.x] = (double)t;
  }
}

// knapsack value / weight excess (builtins.py:258-262)
__device__ __forceinline__ void knap_eval_entry(const void* inst, unsigned off1, int n,
                                                double cap, const short* genes, double* obj,
                                                double* pen) {
  __shared__ double rv[32], rw[32];
  const double* w = (const double*)inst;
  const double* v = (const double*)((const unsigned char*)inst + off1);
  const short* x = genes + (size_t)blockIdx.x * n;
  double sv = 0.0, sw = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sv += v[i] * (double)x[i];
    sw += w[i] * (double)x[i];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    sv += __shfl_xor_sync(0xffffffffu, sv, off);
    sw += __shfl_xor_sync(0xffffffffu, sw, off);
  }
  if ((threadIdx.x & 31) == 0) {
    rv[threadIdx.x >> 5] = sv;
    rw[threadIdx.x >> 5] = sw;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tv = 0.0, tw = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      tv += rv[q];
      tw += rw[q];
    }
    obj[blockIdx.x] = tv;
    const double over = tw - cap;
    pen[blockIdx.x] = over > 0.0 ? over : 0.0;
  }
}

__device__ __forceinline__ void jsp_eval_entry(const void* inst, unsigned off1, int n_jobs,
                                               int per_job, int n_mach, const short* genes,
                                               double* obj) {
  extern __shared__ int jscr[];
  if (threadIdx.x != 0) return;
  JspView J;
  J.mach = (const int*)inst;
  J.dur = (const int*)((const unsigned char*)inst + off1);
  J.n_jobs = n_jobs;
  J.per_job = per_job;
  J.n_mach = n_mach;
  obj[blockIdx.x] = (double)jsp_decode(J, genes + (size_t)blockIdx.x * n_jobs * per_job, jscr);
}

__device__ __forceinline__ void part_eval_entry(const void* inst, go::RowArgs x, const short* genes,
                                                double* obj, double* pen) {
  if (threadIdx.x != 0) return;
  const unsigned char* b = (const unsigned char*)inst;
  PartView v;
  v.dist = (const double*)b;
  v.demand = (const double*)(b + x.off1);
  v.ready = (const double*)(b + x.off2);
  v.due = (const double*)(b + x.off3);
  v.service = (const double*)(b + x.off4);
  v.n = x.n_cells;
  v.d1 = x.d1;
  v.d2 = x.d2;
  v.cap = x.capacity;
  v.tw = x.tw;
  v.variant = x.pvar;
  v.prio = (const double*)(b + x.off2);
  const short* row = genes + (size_t)blockIdx.x * (x.n_cells + x.d1);
  double d, p, o0, o1;
  int veh;
  part_eval(v, row, row + x.n_cells, d, p, &veh);
  part_scal(x, d, veh, &o0, &o1);  // objectives in the problem's order
  obj[(size_t)blockIdx.x * x.mo.m] = o0;
  if (x.mo.m == 2) obj[(size_t)blockIdx.x * 2 + 1] = o1;
  pen[blockIdx.x] = p;
}

// evaluate() of m user-problem rows: one thread per solution (the user objective
// is serial code)
template <class U>
__device__ __forceinline__ void user_eval_entry(const void* inst, int n, int m,
                                                const short* genes, double* obj, double* pen) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const RowSol<short> sol{genes + (size_t)i * n, n};
  const unsigned char* b = (const unsigned char*)inst;
  if (U::kObjectives == 2) {
    obj[2 * i] = U::obj(sol, b);
    obj[2 * i + 1] = U::obj2(sol, b);
  } else {
    obj[i] = U::obj(sol, b);
  }
  pen[i] = U::pen(sol, b);
}

// One application of user operator `slot` to a probe row (register_custom's
// probe, operators.py:646-665): single thread, stream key `key`; the host
// checks the row's validity and the error flag.
template <class U>
__device__ __forceinline__ void user_probe_entry(const void* inst, RowArgs x, int n, int slot,
                                                 unsigned long long key, short* genes, int* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  RowCtx<short> c;
  c.rng.init(key);
  c.row = genes;
  c.full = genes;
  c.mf = x.mf;
  c.d1 = x.mf ? x.d1 : 1;
  c.d2 = x.d2;
  c.n = n;
  c.n_cfg = x.n_cfg;
  c.lb = x.lb;
  c.ub = x.ub;
  short dummy[MAX_RANGES * 2];
  c.rlo = dummy;
  c.rhi = dummy + MAX_RANGES;
  c.rstride = 1;
  c.nr = 0;
  c.err = 0;
  c.mates = nullptr;
  RowOpCtx<short, U> oc{&c,
                        UserScore{(const unsigned char*)inst, x.obj_weight, x.penalty_weight,
                                  x.mo.maxmask, x.w2, x.mo.m},
                        n, c.d1, x.d2, RowInst{(const unsigned char*)inst, x.off1, RI_NONE, 8, n,
                                               x.capacity, n}};
  U::op(slot, oc, (const unsigned char*)inst);
  *err = c.err;
}

// register_custom's probe for a user operator on a BUILT-IN row problem (QAP /
// knapsack / JSP-int: one flat row; partition problems: cells + route sizes),
// one application, single thread, stream key `key`.
template <int KIND, class E, class U>
__device__ __forceinline__ void rowops_probe_entry(const void* inst, RowArgs x, int n, int slot,
                                                   unsigned long long key, short* genes,
                                                   int* err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned char* b = (const unsigned char*)inst;
  if constexpr (KIND == RK_PART) {
    PartCtx c;
    c.rng.init(key);
    c.cells = genes;
    c.sz = genes + x.n_cells;
    c.n = x.n_cells;
    c.d1 = x.d1;
    c.d2 = x.d2;
    c.n_cfg = x.n_cfg;
    c.total = x.n_cells;
    c.err = 0;
    c.mates = nullptr;
    PartView pv;
    pv.dist = (const double*)b;
    pv.demand = (const double*)(b + x.off1);
    pv.ready = (const double*)(b + x.off2);
    pv.due = (const double*)(b + x.off3);
    pv.service = (const double*)(b + x.off4);
    pv.n = x.n_cells;
    pv.d1 = x.d1;
    pv.d2 = x.d2;
    pv.cap = x.capacity;
    pv.tw = x.tw;
    pv.variant = x.pvar;
    pv.prio = (const double*)(b + x.off2);
    PartOpCtx<U> oc{&c, pv, &x, x.penalty_weight, x.n_cells, x.d1, x.d2};
    U::op(slot, oc, b);
    *err = c.err;
  } else {
  RowCtx<short> c;
  c.rng.init(key);
  c.row = genes;
  c.full = genes;
  c.mf = 0;
  c.d1 = 1;
  c.d2 = n;
  c.n = n;
  c.n_cfg = x.n_cfg;
  c.lb = x.lb;
  c.ub = x.ub;
  short dummy[MAX_RANGES * 2];
  c.rlo = dummy;
  c.rhi = dummy + MAX_RANGES;
  c.rstride = 1;
  c.nr = 0;
  c.err = 0;
  c.mates = nullptr;
  const RowInst ri{b, x.off1, KIND == RK_QAP ? RI_QAP : (KIND == RK_KNAP ? RI_KNAP : RI_JSP),
                   KIND == RK_QAP ? (int)sizeof(E) : 8, n, x.capacity, n};
  RowOpCtx<short, U> oc{&c, UserScore{b, x.obj_weight, x.penalty_weight, 0, 0.0, 1}, n, 1, n, ri};
  U::op(slot, oc, b);
  *err = c.err;
  }
}

}  // namespace go

// Kernels of one NVRTC user problem (go_jit.cpp generates `U`); RG: lane rows
// in global memory (a second module, built only for problems that need it).
#define GO_USER_KERNELS(U) GO_USER_KERNELS_RG(U, false)
#define GO_USER_KERNELS_RG(U, RG)                                                             \
  extern "C" __global__ void __launch_bounds__(512, 1) go_evolve_user(go::EvolveArgs a,        \
                                                                      go::RowArgs x) {        \
    go::evolve_row<go::RK_USER, double, short, U, RG>(a, x);                                  \
  }                                                                                           \
  extern "C" __global__ void go_eval_user(const void* inst, int n, int m, const short* g,     \
                                          double* obj, double* pen) {                          \
    go::user_eval_entry<U>(inst, n, m, g, obj, pen);                                          \
  }                                                                                           \
  extern "C" __global__ void go_probe_user_op(const void* inst, go::RowArgs x, int n, int slot, \
                                              unsigned long long key, short* g, int* err) {   \
    go::user_probe_entry<U>(inst, x, n, slot, key, g, err);                                   \
  }

// Kernels of a built-in row problem with NVRTC-compiled user operators
// (register_custom, operators.py:634-669): evolve + probe
#define GO_ROWOPS_KERNELS(KIND, E, G, U, RG)                                                  \
  extern "C" __global__ void __launch_bounds__(512, 1) go_evolve_rowops(go::EvolveArgs a,      \
                                                                        go::RowArgs x) {      \
    go::evolve_row<KIND, E, G, U, RG>(a, x);                                                  \
  }                                                                                           \
  extern "C" __global__ void go_probe_rowop(const void* inst, go::RowArgs x, int n, int slot,  \
                                            unsigned long long key, short* g, int* err) {     \
    go::rowops_probe_entry<KIND, E, U>(inst, x, n, slot, key, g, err);                        \
  }

#define GO_ROW_KERNEL(NAME, KIND, E, G)                                                       \
  extern "C" __global__ void __launch_bounds__(go::row_max_threads(KIND), 1)                   \
      NAME(go::EvolveArgs a, go::RowArgs x) {                                                  \
    go::evolve_row<KIND, E, G>(a, x);                                                         \
  }                                                                                           \
  extern "C" __global__ void __launch_bounds__(go::row_max_threads(KIND), 1)                   \
      NAME##_g(go::EvolveArgs a, go::RowArgs x) {                                              \
    go::evolve_row<KIND, E, G, go::NoUser, true>(a, x);                                       \
  }

// Teams wider than row_max_threads(KIND) (team_size up to 512): the same kernels
// compiled for 512 threads
#define GO_ROW_KERNEL_WIDE(NAME, KIND, E, G)                                                  \
  extern "C" __global__ void __launch_bounds__(512, 1) NAME##_w(go::EvolveArgs a,              \
                                                              go::RowArgs x) {                \
    go::evolve_row<KIND, E, G>(a, x);                                                         \
  }                                                                                           \
  extern "C" __global__ void __launch_bounds__(512, 1) NAME##_gw(go::EvolveArgs a,             \
                                                               go::RowArgs x) {               \
    go::evolve_row<KIND, E, G, go::NoUser, true>(a, x);                                       \
  }
