// go_tsp_entry.cuh — kernel bodies for the TSP path, instantiated both by the
// static library (engine.cu, built-in operators only) and by NVRTC when user
// operators are registered (jit.cpp generates `UserOps`).
#pragma once
#include "go_evolve_perm.cuh"

namespace go {

template <class D, class Custom>
__device__ __forceinline__ void tsp_evolve_entry(const EvolveArgs& a) {
  TspPolicy<StagedView<D>> pol;  // shared-memory layouts are always staged (evolve_perm)
  pol.d.m = (const typename D::Elem*)a.inst;
  pol.d.n = a.n;
  pol.d.sbase = 0;
  pol.d.use_s = 0;
  evolve_perm<TspPolicy<StagedView<D>>, Custom>(a, pol);
}

// evaluate() for m tours (problems.py:77-94 -> builtins.py:67-71)
template <class D>
__device__ __forceinline__ void tsp_eval_entry(const void* inst, int n, const short* genes,
                                               double* obj) {
  typedef typename D::Acc Acc;
  __shared__ Acc red[32];
  TspPolicy<D> pol;
  pol.d.m = (const typename D::Elem*)inst;
  pol.d.n = n;
  pol.d.sbase = 0;
  pol.d.use_s = 0;
  const short* t = genes + (size_t)blockIdx.x * n;
  Acc s = n < 2 ? (Acc)0 : pol.partial(t, n, threadIdx.x, blockDim.x);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    Acc tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    obj[blockIdx.x] = (double)tot;
  }
}

// acceptance_delta for a chain of <= 3 primitive moves, plus the candidate
template <class D>
__device__ __forceinline__ void tsp_delta_entry(const void* inst, int n, const short* genes,
                                                const int* moves, double* delta, short* cand) {
  typedef typename D::Acc Acc;
  extern __shared__ __align__(16) unsigned char dsm[];
  short* row = (short*)dsm;
  __shared__ Chain ch;
  TspPolicy<D> pol;
  pol.d.m = (const typename D::Elem*)inst;
  pol.d.n = n;
  pol.d.sbase = 0;
  pol.d.use_s = 0;
  for (int p = threadIdx.x; p < n; p += blockDim.x) row[p] = genes[(size_t)blockIdx.x * n + p];
  __syncthreads();
  if (threadIdx.x == 0) {
    Chain L;
    L.reset(row, n);
    Acc d = 0;
    for (int s = 0; s < MAX_CHAIN; ++s) {
      const int* mv = moves + ((size_t)blockIdx.x * MAX_CHAIN + s) * 4;
      Move m;
      m.kind = mv[0];
      m.a = mv[1];
      m.b = mv[2];
      m.c = mv[3];
      if (m.kind == MV_NONE) continue;
      unsigned rp = 0, re = 0;
      d += pol.delta(L, m, rp, re);
      L.push(m);
    }
    delta[blockIdx.x] = (double)d;
    ch = L;
  }
  __syncthreads();
  for (int p = threadIdx.x; p < n; p += blockDim.x)
    cand[(size_t)blockIdx.x * n + p] = row[ch.src_all(p)];
}

// registration probe: run one operator once on a probe tour (operators.py:646-665)
template <class D, class Custom>
__device__ __forceinline__ void tsp_probe_entry(const void* inst, int n, int kind,
                                                unsigned long long key, short* genes,
                                                int* err_out) {
  extern __shared__ __align__(16) unsigned char psm[];
  short* row = (short*)psm;
  for (int p = threadIdx.x; p < n; p += blockDim.x) row[p] = genes[p];
  __syncthreads();
  __shared__ Chain ch;
  if (threadIdx.x == 0) {
    TspPolicy<D> pol;
    pol.d.m = (const typename D::Elem*)inst;
    pol.d.n = n;
    pol.d.sbase = 0;
  pol.d.use_s = 0;
    Stream rng;
    rng.init(key);
    Chain L;
    L.reset(row, n);
    PermCtx<TspPolicy<D>> c;
    c.rng = rng;
    c.L = L;
    c.pol = pol;
    c.err = 0;
    c.rd_pos = 0;
    c.rd_elem = 0;
    c.out.kind = MV_NONE;
    run_perm_op<TspPolicy<D>, Custom>(kind, c);
    if (c.out.kind == MV_RELOCATE_BEST) c.out = resolve_relocate_serial(pol, L, c.out.a, c.out.b);
    if (c.out.kind != MV_NONE) L.push(c.out);
    *err_out = c.err;
    ch = L;
  }
  __syncthreads();
  for (int p = threadIdx.x; p < n; p += blockDim.x) genes[p] = row[ch.src_all(p)];
}

}  // namespace go

// Declares the extern "C" kernels of one (layout, custom-ops) instantiation.
// GO_EVOLVE_MAX_THREADS bounds the CTA (teams x lanes) and so the register
// budget per thread (65536 / max threads); the host reads the same value.
#ifndef GO_EVOLVE_MAX_THREADS
#define GO_EVOLVE_MAX_THREADS 512
#endif
#define GO_TSP_KERNELS(SUFFIX, D, CUSTOM)                                                     \
  extern "C" __global__ void __launch_bounds__(GO_EVOLVE_MAX_THREADS, 1)                    \
      go_evolve_tsp_##SUFFIX(go::EvolveArgs a) {                                              \
    go::tsp_evolve_entry<D, CUSTOM>(a);                                                       \
  }                                                                                           \
  extern "C" __global__ void go_probe_tsp_##SUFFIX(const void* inst, int n, int kind,        \
                                                   unsigned long long key, short* genes,      \
                                                   int* err) {                               \
    go::tsp_probe_entry<D, CUSTOM>(inst, n, kind, key, genes, err);                           \
  }
