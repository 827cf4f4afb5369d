// go_perm.cuh — single-row permutation moves as position maps.
//
// A lane never copies the solution (the reference copies it per lane,
// engine.py:570).  Its candidate is the team's current tour composed with
// the <= 3 primitive moves the lane has drawn so far; every move is a map
// src(p) = "position in the pre-move row whose element lands at p":
//
//   SWAP(i,j)          operators.py:205-225 (op_swap)
//   REVERSE(i,j)       operators.py:254-261 (op_reverse), demo 2-opt
//   SEGMENT(s,L,pos)   remove [s,s+L), reinsert at pos of the shortened row:
//                      op_insert (L=1, :228-251), op_or_opt (L=2,3, :264-283),
//                      demo or-opt / node-insert (demo_ops.py:48-89)
//   THREE_OPT(i,j,k,v) row = a b c d with a=[0,i) b=[i,j) c=[j,k) d=[k,n),
//                      reconnected as variant v of op_three_opt (:289-315):
//                      0 a b^r c d, 1 a b c^r d, 2 a b^r c^r d, 3 a c b d,
//                      4 a c b^r d, 5 a c^r b d, 6 a c^r b^r d
//
// Delta evaluation (TSP): a move rewires only the slots (p, p+1 mod n) at its
// cut points; with the symmetric matrices the reference enforces
// (problems.py:97-107) every other edge keeps its length.  The removed edges
// are the cut slots of the OLD row, the added edges the junction slots of the
// NEW row — computing both sets explicitly keeps adjacent / wrap-around /
// whole-row cases exact.  On integer matrices the int64 sum
// equals Φ_ref(cand) − Φ_ref(cur) bit-for-bit.
#pragma once
#include "go_common.cuh"
#include "go_dist.cuh"

namespace go {

enum MoveKind {
  MV_NONE = 0, MV_SWAP = 1, MV_REVERSE = 2, MV_SEGMENT = 3,
  MV_RELOCATE_BEST = 4,  // deferred: SEGMENT(a, b, best slot), resolved cooperatively
  MV_3OPT = 8            // 8 + variant (0..6): THREE_OPT(a=i, b=j, c=k)
};

__device__ __forceinline__ bool is_3opt(int kind) { return kind >= MV_3OPT && kind < MV_3OPT + 7; }

// source position inside [i, k) of three-opt variant v (see header)
__device__ __noinline__ int three_opt_src(int v, int i, int j, int k, int p) {
  const int lc = k - j, q = p - i;
  switch (v) {
    case 0: return p < j ? i + j - 1 - p : p;
    case 1: return p < j ? p : j + k - 1 - p;
    case 2: return p < j ? i + j - 1 - p : j + k - 1 - p;
    case 3: return q < lc ? j + q : i + (q - lc);
    case 4: return q < lc ? j + q : (j - 1) - (q - lc);
    case 5: return q < lc ? (k - 1) - q : i + (q - lc);
    default: return i + k - 1 - p;
  }
}

struct Move {
  int kind, a, b, c;
};

__device__ __forceinline__ int move_src(const Move& m, int p) {
  switch (m.kind) {
    case MV_SWAP:
      return p == m.a ? m.b : (p == m.b ? m.a : p);
    case MV_REVERSE:
      return (p >= m.a && p <= m.b) ? m.a + m.b - p : p;
    case MV_SEGMENT: {
      if (p >= m.c && p < m.c + m.b) return m.a + (p - m.c);
      const int q = p < m.c ? p : p - m.b;
      return q < m.a ? q : q + m.b;
    }
    default:
      if (is_3opt(m.kind) && p >= m.a && p < m.c) return three_opt_src(m.kind - MV_3OPT, m.a, m.b, m.c, p);
      return p;
  }
}

// packed: kind 4 bits | a, b, c 20 bits each (rows up to 2^20 positions)
__device__ __forceinline__ unsigned long long pack_mv(const Move& m) {
  return (unsigned long long)m.kind | ((unsigned long long)(unsigned)m.a << 4) |
         ((unsigned long long)(unsigned)m.b << 24) | ((unsigned long long)(unsigned)m.c << 44);
}
__device__ __forceinline__ Move unpack_mv(unsigned long long v) {
  Move m;
  m.kind = (int)(v & 15u);
  m.a = (int)((v >> 4) & 0xFFFFFu);
  m.b = (int)((v >> 24) & 0xFFFFFu);
  m.c = (int)((v >> 44) & 0xFFFFFu);
  return m;
}

// composed position map of 1..3 packed moves, latest first (out of line:
// it sits behind every at() of a non-empty chain)
__device__ __noinline__ int chain_src(int p, int nm, unsigned long long m0, unsigned long long m1,
                                      unsigned long long m2) {
  if (nm > 2) p = move_src(unpack_mv(m2), p);
  if (nm > 1) p = move_src(unpack_mv(m1), p);
  return move_src(unpack_mv(m0), p);
}

// The lane's candidate: base row (shared memory) composed with <= 3 moves.
struct Chain {
  const i16* base;
  int n, nm;
  unsigned long long pm0, pm1, pm2;  // packed moves

  __device__ __forceinline__ void reset(const i16* b, int n_) {
    base = b;
    n = n_;
    nm = 0;
  }
  __device__ __forceinline__ int src_all(int p) const {
    return nm == 0 ? p : chain_src(p, nm, pm0, pm1, pm2);
  }
  __device__ __forceinline__ int at(int p) const { return base[src_all(p)]; }
  // element at p of the row AFTER applying `mv` on top of this chain
  __device__ __forceinline__ int at_after(const Move& mv, int p) const {
    return at(move_src(mv, p));
  }
  __device__ __forceinline__ void push(const Move& mv) { push_packed(pack_mv(mv)); }
  __device__ __forceinline__ void push_packed(unsigned long long v) {
    if (nm == 0) pm0 = v;
    else if (nm == 1) pm1 = v;
    else pm2 = v;
    ++nm;
  }
};

__device__ __forceinline__ int wrap_slot(int s, int n) { return s < 0 ? s + n : s; }

// old cut slots / new junction slots of a move (deduplicated), see header
__device__ __forceinline__ void move_slots(const Move& mv, int n, int* so, int& no, int* sn,
                                           int& nn) {
  no = nn = 0;
  int a = mv.a, b = mv.b, c = mv.c;
  int o[4], w[4], co = 0, cw = 0;
  if (mv.kind == MV_SWAP) {
    o[0] = w[0] = a - 1;
    o[1] = w[1] = a;
    o[2] = w[2] = b - 1;
    o[3] = w[3] = b;
    co = cw = 4;
  } else if (mv.kind == MV_REVERSE) {
    o[0] = w[0] = a - 1;
    o[1] = w[1] = b;
    co = cw = 2;
  } else if (mv.kind == MV_SEGMENT) {
    if (c == a) return;
    if (c > a) {  // block [a, c+b): old = seg|rest, new = rest|seg
      o[0] = a - 1; o[1] = a + b - 1; o[2] = c + b - 1;
      w[0] = a - 1; w[1] = c - 1;     w[2] = c + b - 1;
    } else {      // block [c, a+b): old = rest|seg, new = seg|rest
      o[0] = c - 1; o[1] = a - 1;     o[2] = a + b - 1;
      w[0] = c - 1; w[1] = c + b - 1; w[2] = a + b - 1;
    }
    co = cw = 3;
  } else if (is_3opt(mv.kind)) {  // cuts i-1, j-1, k-1 -> junctions i-1, i+|first|-1, k-1
    const int first = mv.kind - MV_3OPT < 3 ? b - a : c - b;
    o[0] = a - 1; o[1] = b - 1;         o[2] = c - 1;
    w[0] = a - 1; w[1] = a + first - 1; w[2] = c - 1;
    co = cw = 3;
  }
  for (int i = 0; i < co; ++i) {
    const int s = wrap_slot(o[i], n);
    bool dup = false;
    for (int j = 0; j < no; ++j) dup |= so[j] == s;
    if (!dup) so[no++] = s;
  }
  for (int i = 0; i < cw; ++i) {
    const int s = wrap_slot(w[i], n);
    bool dup = false;
    for (int j = 0; j < nn; ++j) dup |= sn[j] == s;
    if (!dup) sn[nn++] = s;
  }
}

template <class Acc>
struct DeltaOut {
  Acc delta;
  int slots;  // old + new edge slots read (2 positions + 1 element each)
};

// Φ(cand after mv) − Φ(cand) for the cyclic tour objective (builtins.py:67-71).
// Out of line and by value: it has ~16 map-composed reads, and inlining it at
// each call site blew the kernel past the instruction cache.
template <class D>
__device__ __noinline__ DeltaOut<typename D::Acc> tsp_move_delta_ool(const D d, const Chain L,
                                                                     const Move mv) {
  typedef typename D::Acc Acc;
  const int n = L.n;
  int so[4], sn[4], no, nn;
  move_slots(mv, n, so, no, sn, nn);
  Acc delta = 0;
  // one copy of each loop body (code size: move_src is a switch over every
  // move kind and would be inlined once per unrolled slot)
#pragma unroll 1
  for (int i = 0; i < no; ++i) {
    const int p = so[i], q = p + 1 == n ? 0 : p + 1;
    delta -= (Acc)d(L.at(p), L.at(q));
  }
#pragma unroll 1
  for (int i = 0; i < nn; ++i) {
    const int p = sn[i], q = p + 1 == n ? 0 : p + 1;
    delta += (Acc)d(L.at_after(mv, p), L.at_after(mv, q));
  }
  DeltaOut<Acc> o;
  o.delta = delta;
  o.slots = no + nn;
  return o;
}

template <class D>
__device__ __forceinline__ typename D::Acc tsp_move_delta(const D& d, const Chain& L,
                                                          const Move& mv, unsigned& rd_pos,
                                                          unsigned& rd_elem) {
  const DeltaOut<typename D::Acc> o = tsp_move_delta_ool(d, L, mv);
  rd_pos += 2u * (unsigned)o.slots;
  rd_elem += (unsigned)o.slots;
  return o.delta;
}

// ---- operator context (what built-in and user operators may touch) --------
//
// User operator snippets (paper §3.3.2; reference CustomOperator.apply,
// operators.py:79-88) are compiled as
//     template <class Ctx> __device__ void op_<id>(Ctx& ctx) { <snippet> }
// and see exactly this API.  Out-of-range reads or malformed moves set a
// sticky error bit instead of faulting, so the registration probe can
// exclude a broken operator (operators.py:649-665) without killing the run.
// The stream, chain and policy are held BY VALUE: pointers to them (as in
// round 1) pinned all three to the thread's stack, which lives in L2-backed
// local memory here (shared memory takes nearly all of L1), so every draw,
// position read and distance read of an operator paid an L2 round trip.
template <class Policy>
struct PermCtx {
  Stream rng;
  Chain L;
  Policy pol;
  Move out;
  int err;
  unsigned rd_pos, rd_elem;  // algorithmic reads (roofline accounting)

  __device__ __forceinline__ int size() const { return L.n; }
  // branch-free range checks: an out-of-range index reads element 0 and
  // raises the sticky error bit (probe exclusion), never faults
  __device__ __forceinline__ int at(int p) {
    const bool ok = (unsigned)p < (unsigned)L.n;
    err |= ok ? 0 : ERR_OP_RANGE;
    ++rd_pos;
    return L.at(ok ? p : 0);
  }
  __device__ __forceinline__ double dist(int a, int b) {
    const unsigned ni = (unsigned)pol.n_items();
    const bool ok = (unsigned)a < ni && (unsigned)b < ni;
    err |= ok ? 0 : ERR_OP_RANGE;
    ++rd_elem;
    return pol.cost(ok ? a : 0, ok ? b : 0);
  }
  __device__ __forceinline__ double random() { return rng.random(); }
  __device__ __forceinline__ int randbelow(int n) {
    if (n <= 0) {
      err |= ERR_OP_RANGE;
      return 0;
    }
    return rng.randbelow(n);
  }
  __device__ __forceinline__ int randrange(int lo, int hi) {
    if (hi <= lo) {
      err |= ERR_OP_RANGE;
      return lo;
    }
    return rng.randrange(lo, hi);
  }
  __device__ __forceinline__ void swap(int i, int j) {
    const int n = L.n;
    if ((unsigned)i >= (unsigned)n || (unsigned)j >= (unsigned)n || i == j) {
      err |= ERR_OP_MOVE;
      return;
    }
    out.kind = MV_SWAP; out.a = i; out.b = j; out.c = 0;
  }
  __device__ __forceinline__ void reverse(int i, int j) {
    if (i < 0 || j >= L.n || i >= j) {
      err |= ERR_OP_MOVE;
      return;
    }
    out.kind = MV_REVERSE; out.a = i; out.b = j; out.c = 0;
  }
  __device__ __forceinline__ void move_segment(int start, int len, int pos) {
    const int n = L.n;
    if (len < 1 || start < 0 || start + len > n || pos < 0 || pos > n - len) {
      err |= ERR_OP_MOVE;
      return;
    }
    out.kind = MV_SEGMENT; out.a = start; out.b = len; out.c = pos;
  }
  __device__ __forceinline__ void insert(int i, int pos) { move_segment(i, 1, pos); }
  // three-opt reconnection of cuts 0 < i < j < k < n, variant 0..6 (header)
  __device__ __forceinline__ void three_opt(int i, int j, int k, int variant) {
    if (!(0 < i && i < j && j < k && k < L.n) || variant < 0 || variant > 6) {
      err |= ERR_OP_MOVE;
      return;
    }
    out.kind = MV_3OPT + variant; out.a = i; out.b = j; out.c = k;
  }
  // Relocate [start, start+len) to the slot of the shortened row minimising
  //   d(prev, seg[0]) + d(seg[-1], next) - d(prev, next)      (float64)
  // taking the FIRST minimum over slots 0..n-len-1 — exactly the scan of the
  // reference's delta_node_insert (demo_ops.py:71-89, len = 1) and of a
  // full-scan or-opt.  The scan is not run by this lane: the framework
  // resolves every pending relocation of the team with whole warps (32
  // slots per step) after the operators return, so it must be the
  // operator's last action.
  __device__ __forceinline__ void relocate_best(int start, int len) {
    const int n = L.n;
    if (len < 1 || start < 0 || start + len > n || n - len < 2) {
      err |= ERR_OP_MOVE;
      return;
    }
    out.kind = MV_RELOCATE_BEST; out.a = start; out.b = len; out.c = 0;
  }
};

// ---- built-in single-row permutation operators ----------------------------
// Draw order is the reference's; the leading randbelow(1) is _pick_row's
// randrange(len(rows)) over the single row (operators.py:140-144), which
// consumes words in CPython (k = 1, rejection) and therefore here too.
template <class Ctx>
__device__ __forceinline__ void bi_swap(Ctx& c) {
  const int n = c.size();
  if (n < 2) return;
  c.randbelow(1);
  const int i = c.randbelow(n);
  int j = c.randbelow(n - 1);
  j += j >= i;
  c.swap(i, j);
}
template <class Ctx>
__device__ __forceinline__ void bi_insert(Ctx& c) {
  const int n = c.size();
  if (n < 2) return;
  c.randbelow(1);
  const int i = c.randbelow(n);
  const int j = c.randbelow(n);
  c.move_segment(i, 1, j);
}
template <class Ctx>
__device__ __forceinline__ void bi_reverse(Ctx& c) {
  const int n = c.size();
  if (n < 2) return;
  c.randbelow(1);
  const int i = c.randbelow(n - 1);
  const int j = c.randrange(i + 1, n);
  c.reverse(i, j);
}
template <class Ctx>
__device__ __forceinline__ void bi_or_opt(Ctx& c) {
  const int L = c.randrange(2, 4);
  const int n = c.size();
  if (n < L + 1) return;
  c.randbelow(1);
  const int s = c.randbelow(n - L + 1);
  const int pos = c.randbelow(n - L + 1);
  c.move_segment(s, L, pos);
}

// op_three_opt (operators.py:289-315): _pick_row(sol, rng, 4) over the single
// row, sorted sample(range(1, n), 3), variant randrange(7); rows shorter than
// 4 fall back to op_reverse
template <class Ctx>
__device__ __forceinline__ void bi_three_opt(Ctx& c) {
  const int n = c.size();
  if (n < 4) {
    bi_reverse(c);
    return;
  }
  c.randbelow(1);
  int i, j, k;
  sample3_sorted(c, n, i, j, k);
  const int variant = c.randbelow(7);
  c.three_opt(i, j, k, variant);
}

// Serial resolution of a deferred relocation (probe kernel / reference path).
template <class Policy>
__device__ __forceinline__ Move resolve_relocate_serial(const Policy& pol, const Chain& L, int start,
                                                        int len) {
  const int n = L.n, m = n - len;
  const int f = L.at(start), l = L.at(start + len - 1);
  typename Policy::Acc bd = 0;
  int bp = -1;
  for (int pos = 0; pos < m; ++pos) {
    const int qp = pos > 0 ? pos - 1 : m - 1;
    const int prev = L.at(qp < start ? qp : qp + len), nxt = L.at(pos < start ? pos : pos + len);
    const typename Policy::Acc dlt = pol.insertion(prev, f, l, nxt);
    if (bp < 0 || dlt < bd) { bd = dlt; bp = pos; }
  }
  Move mv;
  mv.kind = MV_SEGMENT; mv.a = start; mv.b = len; mv.c = bp;
  return mv;
}

// ---- problem policies over a single permutation row -------------------------
template <class D>
struct TspPolicy {
  typedef typename D::Acc Acc;
  static constexpr bool kIntegral = D::kIntegral;
  // instance staged in shared memory: rows are then at most ~480 long
  static constexpr bool kInSmem = D::kInSmem;
  D d;
  __device__ __forceinline__ int n_items() const { return d.n; }
  __device__ __forceinline__ double cost(int a, int b) const { return (double)d(a, b); }
  __device__ __forceinline__ Acc delta(const Chain& L, const Move& mv, unsigned& rp,
                                       unsigned& re) const {
    return tsp_move_delta(d, L, mv, rp, re);
  }
  // insertion cost of segment (f .. l) between prev and nxt, the reference's
  // float64 expression order (demo_ops.py:62, :83).  On integral matrices the
  // float64 sum of integer terms is exact, so Acc (int64) gives the same value
  // and the same comparisons.
  __device__ __forceinline__ Acc insertion(int prev, int f, int l, int nxt) const {
    if (kIntegral) return (Acc)d(prev, f) + (Acc)d(l, nxt) - (Acc)d(prev, nxt);
    return (Acc)((double)d(prev, f) + (double)d(l, nxt) - (double)d(prev, nxt));
  }
  __device__ __forceinline__ Acc cost_acc(int a, int b) const { return (Acc)d(a, b); }
  typedef typename D::Scan Scan;
  __device__ __forceinline__ Scan cost_scan(int a, int b) const { return (Scan)d(a, b); }
  // full tour length partial sum over slots [lo, hi) step `step` (team reduce)
  __device__ __forceinline__ Acc partial(const i16* t, int n, int lo, int step) const {
    Acc s = 0;
    for (int p = lo; p < n; p += step) s += (Acc)d(t[p], t[p + 1 == n ? 0 : p + 1]);
    return s;
  }
};

}  // namespace go
