// go_init.cuh — device-side population initialisation.
//
// The reference draws K·P random solutions from one MT19937 stream, adds the
// row/column-sum argsort candidates, evaluates the pool and keeps the P best in
// `compare` order (engine.py:252-360).  Here every pool solution owns a Philox
// stream keyed mix64(seed, STREAM_INIT, salt, index), so the K·P draws run one
// solution per thread; the draw order inside a solution is the reference's
// (random.shuffle / randrange, engine.py:252-287), which oracle/engine.py
// restates for the same keys.  Selection is a stable rank: solution i lands in
// slot #{j : j better than i, or equal to i with j < i} — the position a
// stable sort by `compare` (core.py:315-347) gives it.
#pragma once
#include "go_common.cuh"

namespace go {

constexpr u64 STREAM_INIT_ID = 2;  // engine.py:66-71 stream ids (lane, accept, init, ...)

struct InitArgs {
  short* rows;     // [count][W] device rows (to_device_rows layout)
  short* scratch;  // [count][2n + d1] partition work space
  int count, W;
  int kind;        // 0 permutation of n values, 1 partition, 2 cells in [lo, hi]
  int n, d1, d2;   // partition: n values dealt to d1 rows of capacity d2 (W = n + d1)
  int lo, hi;
  int nrows;       // permutation: rows of n values each (MULTI_FIXED)
  u64 seed, salt;
};

__device__ __forceinline__ u64 mix64_4(u64 a, u64 b, u64 c, u64 d) {
  u64 h = 0x9E3779B97F4A7C15ull;
  h = mix64_fold(h, a);
  h = mix64_fold(h, b);
  h = mix64_fold(h, c);
  return mix64_fold(h, d);
}

// random.shuffle (CPython 3.12): for i = n-1 .. 1, j = randbelow(i+1), swap.
__device__ __forceinline__ void shuffle_iota(Stream& s, short* v, int n) {
  for (int i = 0; i < n; ++i) v[i] = (short)i;
  for (int i = n - 1; i > 0; --i) {
    const int j = s.randbelow(i + 1);
    const short t = v[i];
    v[i] = v[j];
    v[j] = t;
  }
}

__global__ void __launch_bounds__(128) init_random_kernel(InitArgs a) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= a.count) return;
  Stream s;
  s.init(mix64_4(a.seed, STREAM_INIT_ID, a.salt, (u64)idx));
  short* row = a.rows + (size_t)idx * a.W;
  if (a.kind == 0) {
    for (int r = 0; r < a.nrows; ++r) shuffle_iota(s, row + r * a.n, a.n);
  } else if (a.kind == 2) {
    const int width = a.hi + 1 - a.lo;
    for (int q = 0; q < a.n; ++q) row[q] = (short)(a.lo + s.randbelow(width));
  } else {
    // engine.py:256-266: shuffle the values, deal each to a uniformly chosen
    // row with room (open rows in row order), appending.
    short* vals = a.scratch + (size_t)idx * (2 * a.n + a.d1);
    short* pick = vals + a.n;
    short* size = pick + a.n;
    shuffle_iota(s, vals, a.n);
    for (int r = 0; r < a.d1; ++r) size[r] = 0;
    int open = a.d1;
    for (int q = 0; q < a.n; ++q) {
      int k = s.randbelow(open);
      int r = 0;
      for (;; ++r)
        if (size[r] < a.d2 && k-- == 0) break;
      pick[q] = (short)r;
      if (++size[r] == a.d2) --open;
    }
    // compact layout: cells in row order, then the sizes
    int at = 0;
    for (int r = 0; r < a.d1; ++r) {
      const int len = size[r];
      row[a.n + r] = (short)len;
      size[r] = (short)at;  // becomes the row cursor
      at += len;
    }
    for (int q = 0; q < a.n; ++q) row[size[pick[q]]++] = vals[q];
  }
}

// compare (core.py:315-347) for one Weighted objective: feasible first, then
// lower penalty, then w·(±obj).
struct InitKey {
  double pen, scal;
};

__device__ __forceinline__ int init_cmp(const InitKey& a, const InitKey& b) {
  const bool fa = a.pen == 0.0, fb = b.pen == 0.0;
  if (fa != fb) return fa ? -1 : 1;
  if (!fa && a.pen != b.pen) return a.pen < b.pen ? -1 : 1;
  if (a.scal == b.scal) return 0;
  return a.scal < b.scal ? -1 : 1;
}

struct SelectArgs {
  const double* obj;  // [M][m_obj]
  const double* pen;  // [M]
  const short* rows;  // [M][W]
  int M, m_obj, W, keep;
  double w;           // scalarisation weight of objective 0
  int maximize;
  int pad;
  short* out_rows;    // [keep][W]
  int* out_idx;       // [keep] pool index of each kept solution
};

__device__ __forceinline__ InitKey init_key(const SelectArgs& a, int i) {
  const double v = a.obj[(size_t)i * a.m_obj];
  return {a.pen[i], 0.0 + a.w * (a.maximize ? -v : v)};
}

__global__ void __launch_bounds__(256) init_select_kernel(SelectArgs a) {
  __shared__ InitKey tile[256];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  InitKey me{0.0, 0.0};
  if (i < a.M) me = init_key(a, i);
  int rank = 0;
  for (int base = 0; base < a.M; base += 256) {
    __syncthreads();
    if (base + (int)threadIdx.x < a.M) tile[threadIdx.x] = init_key(a, base + threadIdx.x);
    __syncthreads();
    const int lim = min(256, a.M - base);
    if (i < a.M)
      for (int t = 0; t < lim; ++t) {
        const int c = init_cmp(tile[t], me);
        rank += (c < 0) | (c == 0 && base + t < i);
      }
  }
  if (i >= a.M || rank >= a.keep) return;
  a.out_idx[rank] = i;
  const short* src = a.rows + (size_t)i * a.W;
  short* dst = a.out_rows + (size_t)rank * a.W;
  for (int q = 0; q < a.W; ++q) dst[q] = src[q];
}

}  // namespace go
