// go_islands.cuh — cross-GPU island exchange (engine.py:483-521 across ranks).
//
// Each rank is one island of the reference's island model.  Every
// `islands.interval` generations a rank exports its top_n members in stable
// best-first order (ties keep the lower member index, exactly the prefix of
// the reference's stable sort) as fixed-size records; the host all-gathers
// the records (NCCL over NVLink on GPUs); every rank then applies the
// reference's migration rule for ITS island on the gathered set:
//   ring          island r receives island r-1's best, replacing its worst
//                 unless the worst is also its best (single member: only if
//                 strictly better)                         (engine.py:494-506)
//   global_top_n  stable top_n of all gathered records replace random
//                 non-best members, drawing from the shared migration stream
//                 mix64(seed, 3, event); ranks below replay their draws so
//                 every island sees the same stream position as in the
//                 single-process loop                       (engine.py:507-519)
// The gathered bests also refresh the global best used by elite injection.
#pragma once
#include "go_args.cuh"
#include "go_common.cuh"
#include "go_epilogue.cuh"

namespace go {

struct IslandArgs {
  int P, W;
  short* genes;
  double* scal;
  double* pen;
  double* obj2;      // [P][2] objective vectors (multi-objective runs) or null
  MoCmp mo;
  short* gbest_genes;
  GlobalState* gs;
  unsigned char* buf;  // records
  int rec_bytes;
  int top_n;
  int n_ranks, rank, strategy;  // strategy 0 ring, 1 global_top_n
  long long event;
  unsigned long long seed;
};

__device__ __forceinline__ double* rec_head(unsigned char* buf, int rec_bytes, int i) {
  return (double*)(buf + (size_t)i * rec_bytes);
}
// record = {scal, pen, o0, o1} header (32 B) + genes
__device__ __forceinline__ short* rec_genes(unsigned char* buf, int rec_bytes, int i) {
  return (short*)(buf + (size_t)i * rec_bytes + 32);
}
__device__ __forceinline__ Cand rec_cand(unsigned char* buf, int rec_bytes, int i) {
  const double* h = rec_head(buf, rec_bytes, i);
  Cand c;
  c.scal = h[0];
  c.pen = h[1];
  c.o0 = h[2];
  c.o1 = h[3];
  c.idx = i;
  return c;
}

__global__ void __launch_bounds__(EPI_THREADS, 1) go_export_elites_kernel(IslandArgs A) {
  __shared__ Cand red[EPI_THREADS / 32];
  __shared__ int s_idx[64];
  const int tn = A.top_n < A.P ? A.top_n : A.P;
  const SolKeys pop{A.pen, A.scal, A.obj2};
  for (int d = 0; d < tn && d < 64; ++d) {
    const Cand b = block_select<false>(pop, 0, A.P, s_idx, d, red, A.mo);
    if (threadIdx.x == 0) {
      s_idx[d] = b.idx;
      double* h = rec_head(A.buf, A.rec_bytes, d);
      h[0] = b.scal;
      h[1] = b.pen;
      h[2] = b.o0;
      h[3] = b.o1;
    }
    copy_genes(rec_genes(A.buf, A.rec_bytes, d), A.genes + (size_t)b.idx * A.W, A.W);
    __syncthreads();
  }
  for (int d = tn; d < A.top_n; ++d) {  // fewer members than top_n: pad with +inf penalty
    if (threadIdx.x == 0) {
      double* h = rec_head(A.buf, A.rec_bytes, d);
      h[0] = 1.7976931348623157e308;
      h[1] = 1.7976931348623157e308;
      h[2] = h[3] = 1.7976931348623157e308;
    }
  }
}

__global__ void __launch_bounds__(EPI_THREADS, 1) go_import_elites_kernel(IslandArgs A) {
  __shared__ Cand red[EPI_THREADS / 32];
  __shared__ int s_sel[64];
  __shared__ int s_slot;
  GlobalState* gs = A.gs;
  const int tn = A.top_n < A.P ? A.top_n : A.P;
  const int nrec = A.n_ranks * A.top_n;

  // refresh the global best from every rank's best record (records d = 0)
  const MoCmp mo = A.mo;
  const SolKeys pop{A.pen, A.scal, A.obj2};
  if (threadIdx.x == 0) {
    int bi = -1;
    Cand best = gbest_cand(gs);
    for (int r = 0; r < A.n_ranks; ++r) {
      const Cand c = rec_cand(A.buf, A.rec_bytes, r * A.top_n);
      if (cand_cmp(c, best, mo) < 0) {
        best = c;
        bi = r * A.top_n;
      }
    }
    s_slot = bi;
    if (bi >= 0) {
      gs->gpen = best.pen;
      gs->gscal = best.scal;
      gs->gobj[0] = best.o0;
      gs->gobj[1] = best.o1;
      gs->gev = -1;
    }
  }
  __syncthreads();
  if (s_slot >= 0) copy_genes(A.gbest_genes, rec_genes(A.buf, A.rec_bytes, s_slot), A.W);
  __syncthreads();

  if (A.n_ranks < 2) return;
  if (A.strategy == 0) {  // ring: donor = previous rank's best
    const int src = ((A.rank - 1 + A.n_ranks) % A.n_ranks) * A.top_n;
    const Cand h = rec_cand(A.buf, A.rec_bytes, src);
    if (A.P == 1) {
      if (cand_cmp(h, pop.at(0), mo) < 0)
        put_solution_raw(A.genes, A.scal, A.pen, A.obj2, A.W, 0,
                         rec_genes(A.buf, A.rec_bytes, src), h);
      return;
    }
    const Cand w = block_select<true>(pop, 0, A.P, nullptr, 0, red, mo);
    const Cand b = block_select<false>(pop, 0, A.P, nullptr, 0, red, mo);
    if (w.idx != b.idx)
      put_solution_raw(A.genes, A.scal, A.pen, A.obj2, A.W, w.idx,
                       rec_genes(A.buf, A.rec_bytes, src), h);
    return;
  }
  // global_top_n: stable top tn over the gathered records (rank-major order)
  if (threadIdx.x == 0) {
    int nsel = 0;
    for (int d = 0; d < tn && d < 64; ++d) {
      int bi = -1;
      for (int i = 0; i < nrec; ++i) {
        bool taken = false;
        for (int q = 0; q < nsel; ++q) taken |= s_sel[q] == i;
        if (taken) continue;
        const Cand h = rec_cand(A.buf, A.rec_bytes, i);
        if (h.pen == 1.7976931348623157e308) continue;  // padding
        if (bi < 0) {
          bi = i;
          continue;
        }
        if (cand_cmp(h, rec_cand(A.buf, A.rec_bytes, bi), mo) < 0) bi = i;
      }
      if (bi < 0) break;
      s_sel[nsel++] = bi;
    }
    s_slot = nsel;
  }
  __syncthreads();
  const int nd = s_slot;
  const Cand b = block_select<false>(pop, 0, A.P, nullptr, 0, red, mo);
  const int nslots = A.P - 1;
  Stream mr;
  mr.init(mix64_3(A.seed, 3, (u64)A.event));
  // replay the draws of islands 0 .. rank-1 (same sizes, same donor count)
  if (nslots > 0)
    for (int r = 0; r < A.rank; ++r)
      for (int d = 0; d < nd; ++d) mr.randbelow(nslots);
  for (int d = 0; d < nd; ++d) {
    if (nslots <= 0) break;
    __shared__ int s_dst;
    if (threadIdx.x == 0) {
      int s = mr.randbelow(nslots);
      if (s >= b.idx) ++s;
      s_dst = s;
    }
    __syncthreads();
    put_solution_raw(A.genes, A.scal, A.pen, A.obj2, A.W, s_dst,
                     rec_genes(A.buf, A.rec_bytes, s_sel[d]),
                     rec_cand(A.buf, A.rec_bytes, s_sel[d]));
    __syncthreads();
  }
}

}  // namespace go
