// engine.cu — libcugenopt.so: the C ABI (include/cugenopt.h) over the
// hand-written sm_100a kernels in kernels/*.cuh.
//
// Host responsibilities (all native, no Python on the run path):
//   * instance analysis + layout choice (go_dist.cuh) and device images;
//   * shared-memory auto-extension: cudaFuncSetAttribute up to the device's
//     opt-in limit (paper §4.3), teams-per-CTA from the remaining budget;
//   * the generation loop of _run_single (engine.py:681-750) as a pipeline of
//     (evolve chunk, epilogue) launches that never waits on the device except
//     to bound the queue depth; wall-clock budget enforced on the device;
//   * NVRTC-compiled user operators (go_jit.cpp) with probe/exclusion.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/cugenopt.h"
#include "go_drv.h"
#include "go_jit.h"
#include "kernels/go_epilogue.cuh"
#include "kernels/go_init.cuh"
#include "kernels/go_islands.cuh"
#include "kernels/go_row_entry.cuh"
#include "kernels/go_tsp_entry.cuh"

// ---- static instantiations: built-in operators, every layout ----------------
GO_TSP_KERNELS(i16f, go::DistI16Full, go::NoCustomOps)
GO_TSP_KERNELS(i16t, go::DistI16Tri, go::NoCustomOps)
GO_TSP_KERNELS(i32f, go::DistI32Full, go::NoCustomOps)
GO_TSP_KERNELS(i32t, go::DistI32Tri, go::NoCustomOps)
GO_TSP_KERNELS(f64f, go::DistF64Full, go::NoCustomOps)
GO_TSP_KERNELS(f64t, go::DistF64Tri, go::NoCustomOps)
GO_TSP_KERNELS(i16g, go::DistI16FullG, go::NoCustomOps)
GO_TSP_KERNELS(i32g, go::DistI32FullG, go::NoCustomOps)
GO_TSP_KERNELS(f64g, go::DistF64FullG, go::NoCustomOps)

#define GO_EVAL_KERNELS(SUFFIX, D)                                                            \
  extern "C" __global__ void go_eval_tsp_##SUFFIX(const void* inst, int n, const short* g,   \
                                                  double* obj) {                             \
    go::tsp_eval_entry<D>(inst, n, g, obj);                                                   \
  }                                                                                           \
  extern "C" __global__ void go_delta_tsp_##SUFFIX(const void* inst, int n, const short* g,  \
                                                   const int* mv, double* d, short* cand) {   \
    go::tsp_delta_entry<D>(inst, n, g, mv, d, cand);                                          \
  }
GO_EVAL_KERNELS(i16, go::DistI16FullG)
GO_EVAL_KERNELS(i32, go::DistI32FullG)
GO_EVAL_KERNELS(f64, go::DistF64FullG)

// ---- row family: QAP / knapsack / JSP-int -------------------------------------
GO_ROW_KERNEL(go_evolve_qap_i16, go::RK_QAP, short, short)
GO_ROW_KERNEL(go_evolve_qap_i32, go::RK_QAP, int, short)
GO_ROW_KERNEL(go_evolve_qap_f64, go::RK_QAP, double, short)
GO_ROW_KERNEL(go_evolve_knap, go::RK_KNAP, double, unsigned char)
GO_ROW_KERNEL(go_evolve_jsp, go::RK_JSP, int, short)
GO_ROW_KERNEL(go_evolve_part, go::RK_PART, double, short)
GO_ROW_KERNEL_WIDE(go_evolve_knap, go::RK_KNAP, double, unsigned char)
GO_ROW_KERNEL_WIDE(go_evolve_jsp, go::RK_JSP, int, short)
GO_ROW_KERNEL_WIDE(go_evolve_part, go::RK_PART, double, short)
extern "C" __global__ void go_eval_part(const void* inst, go::RowArgs x, const short* g, double* obj,
                                        double* pen) {
  go::part_eval_entry(inst, x, g, obj, pen);
}
extern "C" __global__ void go_eval_qap_i16(const void* inst, unsigned off1, int n, const short* g,
                                           double* obj) {
  go::qap_eval_entry<short>(inst, off1, n, g, obj);
}
extern "C" __global__ void go_eval_qap_i32(const void* inst, unsigned off1, int n, const short* g,
                                           double* obj) {
  go::qap_eval_entry<int>(inst, off1, n, g, obj);
}
extern "C" __global__ void go_eval_qap_f64(const void* inst, unsigned off1, int n, const short* g,
                                           double* obj) {
  go::qap_eval_entry<double>(inst, off1, n, g, obj);
}
extern "C" __global__ void go_eval_knap(const void* inst, unsigned off1, int n, double cap,
                                        const short* g, double* obj, double* pen) {
  go::knap_eval_entry(inst, off1, n, cap, g, obj, pen);
}
extern "C" __global__ void go_eval_jsp(const void* inst, unsigned off1, int n_jobs, int per_job,
                                       int n_mach, const short* g, double* obj) {
  go::jsp_eval_entry(inst, off1, n_jobs, per_job, n_mach, g, obj);
}

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess)                                                                  \
      return fail(GO_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));              \
  } while (0)

#define CU(x)                                                                               \
  do {                                                                                      \
    if (!gohost::drv()) return fail(GO_E_NODEVICE, "CUDA driver API unavailable");          \
    CUresult r_ = (x);                                                                      \
    if (r_ != CUDA_SUCCESS) {                                                               \
      const char* s_ = nullptr;                                                             \
      gohost::drv()->GetErrorString(r_, &s_);                                               \
      return fail(GO_E_CUDA, std::string(#x) + ": " + (s_ ? s_ : "?"));                     \
    }                                                                                       \
  } while (0)

enum Elem { E_I16 = 0, E_I32 = 1, E_F64 = 2 };

struct LayoutInfo {
  const char* dist_type;  // device type name (NVRTC instantiation)
  void* evolve;
  void* probe;
  int elem;
  bool tri, global;
};

const LayoutInfo kLayouts[9] = {
    {"go::DistI16Full", (void*)go_evolve_tsp_i16f, (void*)go_probe_tsp_i16f, E_I16, false, false},
    {"go::DistI16Tri", (void*)go_evolve_tsp_i16t, (void*)go_probe_tsp_i16t, E_I16, true, false},
    {"go::DistI32Full", (void*)go_evolve_tsp_i32f, (void*)go_probe_tsp_i32f, E_I32, false, false},
    {"go::DistI32Tri", (void*)go_evolve_tsp_i32t, (void*)go_probe_tsp_i32t, E_I32, true, false},
    {"go::DistF64Full", (void*)go_evolve_tsp_f64f, (void*)go_probe_tsp_f64f, E_F64, false, false},
    {"go::DistF64Tri", (void*)go_evolve_tsp_f64t, (void*)go_probe_tsp_f64t, E_F64, true, false},
    {"go::DistI16FullG", (void*)go_evolve_tsp_i16g, (void*)go_probe_tsp_i16g, E_I16, false, true},
    {"go::DistI32FullG", (void*)go_evolve_tsp_i32g, (void*)go_probe_tsp_i32g, E_I32, false, true},
    {"go::DistF64FullG", (void*)go_evolve_tsp_f64g, (void*)go_probe_tsp_f64g, E_F64, false, true},
};

size_t elem_size(int e) { return e == E_I16 ? 2 : (e == E_I32 ? 4 : 8); }

int global_layout(int elem) { return 6 + elem; }

unsigned pad16(size_t b) { return (unsigned)((b + 15) / 16 * 16); }

struct DeviceInfo {
  int sm = 0, smem_optin = 0, l2 = 0;
};

int query_device(int dev, DeviceInfo* di) {
  CK(cudaDeviceGetAttribute(&di->sm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&di->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  CK(cudaDeviceGetAttribute(&di->l2, cudaDevAttrL2CacheSize, dev));
  return GO_OK;
}

unsigned team_bytes_for(int elem, int n, int TS) {
  return elem == E_F64 ? go::PermSmem::team_bytes<double>(n, TS)
                       : go::PermSmem::team_bytes<long long>(n, TS);
}

// smem bytes needed by one CTA with E teams for a given layout
size_t cta_smem(int layout, int n, int E, int TS, size_t inst_img_bytes) {
  const LayoutInfo& L = kLayouts[layout];
  const unsigned inst = L.global ? 0u : pad16(inst_img_bytes);
  return go::PermSmem::team_off(inst) + (size_t)E * team_bytes_for(L.elem, n, TS);
}

}  // namespace

constexpr size_t kStackBytes = 4096;

// ---- handles -------------------------------------------------------------------
struct go_problem {
  int kind = 0, n = 0, d1 = 1, d2 = 0, device = 0;
  int family = 0;          // 0: TSP (chain kernel), 1: row kernel
  // row family
  int row_kind = 0;        // go::RowKind
  void* d_img = nullptr;   // instance image
  size_t img_bytes = 0;
  unsigned off1 = 0;
  double capacity = 0.0;
  int n_jobs = 0, per_job = 0, n_mach = 0, lb = 0, ub = 0, scratch_ints = 0, gsize = 2;
  // partition problems: stored compactly as cells[n_cells] + sizes[d1] (n = n_cells + d1)
  int n_cells = 0, tw = 0;
  unsigned off2 = 0, off3 = 0, off4 = 0;
  int elem = E_F64;
  bool integral = false;
  void* d_full = nullptr;  // n*n in elem type (global reads, eval kernels)
  void* d_tri = nullptr;   // packed strict upper triangle (smem image)
  size_t full_bytes = 0, tri_bytes = 0;
  DeviceInfo dev;
  // routing objectives (n_obj 1 or 2; kinds 0 distance, 1 vehicles)
  int n_obj = 1, okind0 = 0, okind1 = 1;
  int pvar = 0;  // partition variant (RowArgs::pvar)
  // user problems (RK_USER): NVRTC objective module, encoding
  gohost::JitModule user_mod;
  gohost::JitModule user_mod_g;  // lane rows in global memory, built when first needed
  gohost::UserProblemSrc user_src;  // kept to rebuild the module with user operators
  int enc = 0;
  int mf = 0;  // MULTI_FIXED user rows: 1 permutation rows, 2 binary / integer cells
  // user operators
  std::vector<gohost::UserOpSrc> ops;  // registered (compiled and probed)
  std::map<int, gohost::JitModule> jit;  // per layout
};

struct go_engine {
  go_problem* prob = nullptr;
  go_engine_config cfg{};
  int P = 0, T = 0, TS = 0, E = 0, n = 0, W = 0, layout = 0;
  unsigned inst_bytes = 0;
  const void* inst = nullptr;
  size_t smem = 0;
  int grid = 0;
  cudaStream_t stream = nullptr;
  void* k_evolve = nullptr;
  CUfunction k_evolve_jit = nullptr;
  // device state
  short *genes = nullptr, *best_genes = nullptr, *gbest_genes = nullptr, *scratch = nullptr;
  double *scal = nullptr, *pen = nullptr, *best_scal = nullptr, *best_pen = nullptr;
  long long* best_gen = nullptr;
  int *usage = nullptr, *impr = nullptr, *k_usage = nullptr, *k_impr = nullptr;
  long long* agg = nullptr;
  double *rec_scal = nullptr, *rec_pen = nullptr;
  double* temps = nullptr;  // ring [kDepth][MAX_CHUNK]
  double* h_temps = nullptr;
  go::RegistryDev* reg = nullptr;
  go::GlobalState* gs = nullptr;
  double* history = nullptr;
  long long hist_cap = 0;
  bool history_on = false;
  int* h_stop = nullptr;
  int* d_stop_map = nullptr;
  long long gen_enqueued = 0;
  double obj_sign_over_w = 1.0;
  int nseq = 0;
  int teams_per_sm = 0;
  // crossover snapshot (EvolveArgs::snap): allocated when the registry holds
  // OX / uniform crossover; `coop` = the grid fits one co-resident wave, so a
  // chunk may span generations (grid barrier), else chunks are 1 generation
  short* snap = nullptr;  // [SNAP_DEPTH][P][W]
  int* prog = nullptr;     // [P] published snapshot generation per team
  short* lane_rows = nullptr;  // TSP whole-row operators: [P][T][2][n]
  // objective vectors (multi-objective / Lexicographic runs): [P][2], [P][2], [MAX_CHUNK][P][2]
  double *obj2 = nullptr, *best_obj2 = nullptr, *rec_obj2 = nullptr;
  go::MoCmp mo{};
  bool xover = false, coop = false;
  static const int kDepth = 8;
  cudaEvent_t ring_ev[kDepth] = {};
  cudaEvent_t k_beg[kDepth] = {}, k_end[kDepth] = {};  // evolve-kernel-only timing
  bool k_pending[kDepth] = {};
  cudaEvent_t t_start = nullptr, t_stop = nullptr;
  long long launches = 0;
  // pinned host staging of go_engine_set/get_population (grown on demand);
  // pin_ev marks the last copy out of it on `stream`
  unsigned char* h_pin = nullptr;
  size_t h_pin_bytes = 0;
  cudaEvent_t pin_ev = nullptr;
};

extern "C" {

int go_abi_version(void) { return GO_ABI_VERSION; }

const char* go_last_error(void) { return g_err.c_str(); }

int go_device_count(int* count) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess || c == 0) {
    *count = 0;
    return fail(GO_E_NODEVICE, std::string("no CUDA device: ") + cudaGetErrorString(e));
  }
  *count = c;
  return GO_OK;
}

int go_device_query(int device, go_device_info* out) {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, device));
  DeviceInfo di;
  int rc = query_device(device, &di);
  if (rc) return rc;
  memset(out, 0, sizeof(*out));
  out->device = device;
  out->sm_count = di.sm;
  out->max_smem_optin = di.smem_optin;
  out->l2_bytes = di.l2;
  out->cc_major = p.major;
  out->cc_minor = p.minor;
  out->global_mem = (int64_t)p.totalGlobalMem;
  snprintf(out->name, sizeof(out->name), "%s", p.name);
  return GO_OK;
}

static int create_row_problem(const go_problem_desc* d, int device, go_problem** out);

int go_problem_create(const go_problem_desc* d, int device, go_problem** out) {
  if (!d || !out) return fail(GO_E_INVALID, "null argument");
  if (d->kind == GO_QAP || d->kind == GO_KNAPSACK || d->kind == GO_JSP_INT ||
      d->kind == GO_VRPTW || d->kind == GO_CVRP || d->kind == GO_VRP_PRIORITY ||
      d->kind == GO_VRP_NONLINEAR)
    return create_row_problem(d, device, out);
  if (d->kind != GO_TSP)
    return fail(GO_E_UNSUPPORTED, "problem kind " + std::to_string(d->kind) +
                                      " has no device path in this build");
  const int n = d->n;
  if (n < 1 || n > 32767) return fail(GO_E_INVALID, "TSP size must be in [1, 32767]");
  if (!d->dist) return fail(GO_E_INVALID, "TSP needs a distance matrix");
  // check_distance_matrix (problems.py:97-107): square, >= 0, zero diagonal, symmetric
  bool integral = true;
  double maxv = 0;
  for (int i = 0; i < n; ++i) {
    if (d->dist[(size_t)i * n + i] != 0.0)
      return fail(GO_E_INVALID, "distance matrix must have a zero diagonal");
    for (int j = 0; j < n; ++j) {
      const double v = d->dist[(size_t)i * n + j];
      if (!(v >= 0.0) || !std::isfinite(v))
        return fail(GO_E_INVALID, "distance matrix must be nonnegative and finite");
      if (v != d->dist[(size_t)j * n + i])
        return fail(GO_E_INVALID, "distance matrix declared symmetric but is not");
      if (v != std::floor(v)) integral = false;
      maxv = std::max(maxv, v);
    }
  }
  if (maxv > 2147483647.0) integral = false;
  std::unique_ptr<go_problem> p(new go_problem());
  p->kind = GO_TSP;
  p->n = n;
  p->d1 = 1;
  p->d2 = n;
  p->device = device;
  p->integral = integral;
  p->elem = integral ? (maxv <= 32767.0 ? E_I16 : E_I32) : E_F64;
  CK(cudaSetDevice(device));
  CK(cudaFree(0));
  int rc = query_device(device, &p->dev);
  if (rc) return rc;
  const size_t es = elem_size(p->elem);
  p->full_bytes = (size_t)n * n * es;
  p->tri_bytes = (size_t)n * (n - 1) / 2 * es;
  std::vector<unsigned char> full(pad16(p->full_bytes)), tri(pad16(std::max<size_t>(p->tri_bytes, 16)));
  size_t t = 0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double v = d->dist[(size_t)i * n + j];
      const size_t at = (size_t)i * n + j;
      if (p->elem == E_I16) ((short*)full.data())[at] = (short)v;
      else if (p->elem == E_I32) ((int*)full.data())[at] = (int)v;
      else ((double*)full.data())[at] = v;
      if (j > i) {
        if (p->elem == E_I16) ((short*)tri.data())[t] = (short)v;
        else if (p->elem == E_I32) ((int*)tri.data())[t] = (int)v;
        else ((double*)tri.data())[t] = v;
        ++t;
      }
    }
  CK(cudaMalloc(&p->d_full, full.size()));
  CK(cudaMemcpy(p->d_full, full.data(), full.size(), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&p->d_tri, tri.size()));
  CK(cudaMemcpy(p->d_tri, tri.data(), tri.size(), cudaMemcpyHostToDevice));
  *out = p.release();
  return GO_OK;
}

static int create_row_problem(const go_problem_desc* d, int device, go_problem** out) {
  std::unique_ptr<go_problem> p(new go_problem());
  p->kind = d->kind;
  p->family = 1;
  p->device = device;
  CK(cudaSetDevice(device));
  CK(cudaFree(0));
  int rc = query_device(device, &p->dev);
  if (rc) return rc;
  std::vector<unsigned char> img;
  if (d->kind == GO_QAP) {  // builtins.py:265-290
    const int n = d->n;
    if (n < 1 || n > 32767 || !d->flow || !d->dist) return fail(GO_E_INVALID, "QAP needs n, flow, dist");
    bool integral = true;
    double maxv = 0;
    for (size_t i = 0; i < (size_t)n * n; ++i) {
      for (const double v : {d->flow[i], d->dist[i]}) {
        if (!std::isfinite(v)) return fail(GO_E_INVALID, "QAP matrices must be finite");
        if (v != std::floor(v)) integral = false;
        maxv = std::max(maxv, std::fabs(v));
      }
    }
    p->elem = !integral ? E_F64 : (maxv <= 32767.0 ? E_I16 : (maxv <= 2147483647.0 ? E_I32 : E_F64));
    const size_t es = elem_size(p->elem), mb = (size_t)n * n * es;
    p->off1 = pad16(mb);
    img.assign(p->off1 + pad16(mb), 0);
    for (size_t i = 0; i < (size_t)n * n; ++i) {
      const double f = d->flow[i], v = d->dist[i];
      if (p->elem == E_I16) {
        ((short*)img.data())[i] = (short)f;
        ((short*)(img.data() + p->off1))[i] = (short)v;
      } else if (p->elem == E_I32) {
        ((int*)img.data())[i] = (int)f;
        ((int*)(img.data() + p->off1))[i] = (int)v;
      } else {
        ((double*)img.data())[i] = f;
        ((double*)(img.data() + p->off1))[i] = v;
      }
    }
    p->n = n;
    p->row_kind = go::RK_QAP;
    p->gsize = 2;
  } else if (d->kind == GO_KNAPSACK) {  // builtins.py:240-262
    const int n = d->n;
    if (n < 1 || n > 32767 || !d->weights || !d->values) return fail(GO_E_INVALID, "knapsack needs n, weights, values");
    p->off1 = pad16((size_t)n * 8);
    img.assign(2 * (size_t)p->off1, 0);
    memcpy(img.data(), d->weights, (size_t)n * 8);
    memcpy(img.data() + p->off1, d->values, (size_t)n * 8);
    p->capacity = d->capacity;
    p->n = n;
    p->row_kind = go::RK_KNAP;
    p->gsize = 1;
    p->ub = 1;
  } else if (d->kind == GO_VRPTW || d->kind == GO_CVRP || d->kind == GO_VRP_PRIORITY ||
             d->kind == GO_VRP_NONLINEAR) {  // builtins.py:80-237
    const int n = d->n, v = d->d1;
    if (n < 1 || n > 30000 || v < 1 || v > 2000 || !d->dist || !d->demands)
      return fail(GO_E_INVALID, "routing needs n customers, vehicles, dist (n+1)^2, demands");
    const bool tw = d->kind == GO_VRPTW;
    if (tw && (!d->ready || !d->due || !d->service)) return fail(GO_E_INVALID, "VRPTW needs ready/due/service");
    const size_t n1 = (size_t)n + 1;
    p->off1 = pad16(n1 * n1 * 8);
    p->off2 = p->off1 + pad16((size_t)n * 8);
    p->off3 = p->off2 + pad16(n1 * 8);
    p->off4 = p->off3 + pad16(n1 * 8);
    img.assign(p->off4 + pad16(n1 * 8), 0);
    memcpy(img.data(), d->dist, n1 * n1 * 8);
    memcpy(img.data() + p->off1, d->demands, (size_t)n * 8);
    if (tw) {
      memcpy(img.data() + p->off2, d->ready, n1 * 8);
      memcpy(img.data() + p->off3, d->due, n1 * 8);
      memcpy(img.data() + p->off4, d->service, n1 * 8);
    }
    p->pvar = d->kind == GO_VRP_PRIORITY ? 1 : (d->kind == GO_VRP_NONLINEAR ? 2 : 0);
    if (p->pvar == 1) {  // priorities in the (unused) ready-time slot
      if (!d->priorities) return fail(GO_E_INVALID, "vrp_priority needs priorities");
      memcpy(img.data() + p->off2, d->priorities, (size_t)n * 8);
    }
    p->capacity = d->capacity;
    p->tw = tw;
    p->n_cells = n;
    p->n_obj = d->n_obj == 2 ? 2 : 1;
    p->okind0 = d->obj_kind[0] == 1 ? 1 : 0;
    p->okind1 = d->obj_kind[1] == 0 ? 0 : 1;
    if (d->n_obj < 0 || d->n_obj > 2) return fail(GO_E_UNSUPPORTED, "routing supports 1 or 2 objectives");
    p->row_kind = go::RK_PART;
    p->gsize = 2;
    p->n = n + v;  // compact row length
    p->d1 = v;
    p->d2 = d->d2 > 0 ? d->d2 : n;
  } else {  // GO_JSP_INT, builtins.py:408-456
    const int nj = d->n_jobs, pj = d->ops_per_job;
    if (nj < 1 || pj < 1 || nj > 255 * 4 || (long long)nj * pj > 32767 || !d->jsp_machine || !d->jsp_duration)
      return fail(GO_E_INVALID, "JSP needs jobs x ops (<= 32767 operations)");
    const int n = nj * pj;
    int nm = 0;
    for (int i = 0; i < n; ++i) {
      if (d->jsp_machine[i] < 0 || d->jsp_duration[i] < 0) return fail(GO_E_INVALID, "negative JSP entry");
      nm = std::max(nm, d->jsp_machine[i] + 1);
    }
    if (pj > 255) return fail(GO_E_UNSUPPORTED, "more than 255 operations per job");
    p->off1 = pad16((size_t)n * 4);
    img.assign(2 * (size_t)p->off1, 0);
    memcpy(img.data(), d->jsp_machine, (size_t)n * 4);
    memcpy(img.data() + p->off1, d->jsp_duration, (size_t)n * 4);
    p->n = n;
    p->n_jobs = nj;
    p->per_job = pj;
    p->n_mach = nm;
    p->lb = 0;
    p->ub = n - 1;
    p->row_kind = go::RK_JSP;
    p->gsize = 2;
    p->scratch_ints = go::jsp_scratch_ints(nj, nm);
  }
  if (p->row_kind != go::RK_PART) {
    p->d1 = 1;
    p->d2 = p->n;
  }
  p->img_bytes = img.size();
  CK(cudaMalloc(&p->d_img, img.size()));
  CK(cudaMemcpy(p->d_img, img.data(), img.size(), cudaMemcpyHostToDevice));
  *out = p.release();
  return GO_OK;
}

static bool c_identifier(const char* s) {
  if (!s || !*s || !(std::isalpha((unsigned char)*s) || *s == '_')) return false;
  for (const char* c = s; *c; ++c)
    if (!(std::isalnum((unsigned char)*c) || *c == '_')) return false;
  return std::strlen(s) < 64;
}

int go_problem_create_user(const go_user_problem_desc* d, int device, go_problem** out, char* log,
                           int log_len) {
  if (!d || !out || !d->compute_obj) return fail(GO_E_INVALID, "user problem needs compute_obj");
  if (d->encoding < 0 || d->encoding > 2) return fail(GO_E_INVALID, "encoding must be 0, 1 or 2");
  if (d->n < 1 || d->n > 32767) return fail(GO_E_INVALID, "n must be in [1, 32767]");
  if (d->encoding == 2 && (d->lb > d->ub || d->lb < 0 || d->ub > 32767))
    return fail(GO_E_INVALID, "integer bounds must satisfy 0 <= lb <= ub <= 32767");
  if (d->n_data < 0 || (d->n_data > 0 && (!d->data_names || !d->data || !d->data_lens)))
    return fail(GO_E_INVALID, "data arrays need names, pointers and lengths");
  std::unique_ptr<go_problem> p(new go_problem());
  p->kind = GO_USER;
  p->family = 1;
  p->device = device;
  CK(cudaSetDevice(device));
  CK(cudaFree(0));
  int rc = query_device(device, &p->dev);
  if (rc) return rc;
  gohost::UserProblemSrc up;
  up.obj = d->compute_obj;
  up.pen = d->compute_penalty ? d->compute_penalty : "";
  up.obj2 = d->compute_obj2 ? d->compute_obj2 : "";
  std::vector<unsigned char> img;
  for (int i = 0; i < d->n_data; ++i) {
    if (!c_identifier(d->data_names[i]) || d->data_lens[i] < 0 ||
        (d->data_lens[i] > 0 && !d->data[i]))
      return fail(GO_E_INVALID, std::string("bad data array #") + std::to_string(i));
    for (int j = 0; j < i; ++j)
      if (std::strcmp(d->data_names[i], d->data_names[j]) == 0)
        return fail(GO_E_INVALID, std::string("duplicate data name ") + d->data_names[i]);
    const size_t off = img.size(), bytes = (size_t)d->data_lens[i] * 8;
    img.resize(off + pad16(bytes), 0);
    if (bytes) memcpy(img.data() + off, d->data[i], bytes);
    up.names.push_back(d->data_names[i]);
    up.offsets.push_back(off);
    up.lens.push_back(d->data_lens[i]);
  }
  if (img.empty()) img.assign(16, 0);
  const int rows = d->rows > 1 ? d->rows : 1;
  if ((long long)rows * d->n > 32767) return fail(GO_E_INVALID, "rows * n must be <= 32767");
  p->n = rows * d->n;  // device row: the d1 x d2 genes, row-major
  p->d1 = rows;
  p->d2 = d->n;
  p->mf = rows > 1 ? (d->encoding == 0 ? 1 : 2) : 0;
  p->n_obj = d->compute_obj2 ? 2 : 1;
  p->enc = d->encoding;
  p->lb = d->encoding == 0 ? 0 : (d->encoding == 1 ? 0 : d->lb);
  p->ub = d->encoding == 0 ? d->n - 1 : (d->encoding == 1 ? 1 : d->ub);
  p->row_kind = go::RK_USER;
  p->gsize = 2;
  p->img_bytes = img.size();
  std::string jlog;
  p->user_src = up;
  rc = gohost::jit_build_user(up, &p->user_mod, &jlog);
  if (log && log_len > 0) {
    std::strncpy(log, jlog.c_str(), (size_t)log_len - 1);
    log[log_len - 1] = 0;
  }
  if (rc) return fail(rc, "NVRTC build of the user problem failed: " + jlog.substr(0, 2000));
  CK(cudaMalloc(&p->d_img, img.size()));
  CK(cudaMemcpy(p->d_img, img.data(), img.size(), cudaMemcpyHostToDevice));
  *out = p.release();
  return GO_OK;
}

int go_problem_destroy(go_problem* p) {
  if (!p) return GO_OK;
  cudaSetDevice(p->device);
  cudaFree(p->d_img);
  for (auto& kv : p->jit)
    if (kv.second.mod && gohost::drv()) gohost::drv()->ModuleUnload(kv.second.mod);
  if (p->user_mod.mod && gohost::drv()) gohost::drv()->ModuleUnload(p->user_mod.mod);
  if (p->user_mod_g.mod && gohost::drv()) gohost::drv()->ModuleUnload(p->user_mod_g.mod);
  cudaFree(p->d_full);
  cudaFree(p->d_tri);
  delete p;
  return GO_OK;
}

}  // extern "C"

namespace {

// thread cap of the JIT TSP module for a team stride: the default launch
// bound (jit_max_threads) unless one team alone needs more
int tsp_jit_cap(int TS) { return std::max(gohost::jit_max_threads(), TS); }

// Layout + teams-per-CTA choice (paper §4.3 three-layer split: the problem
// states its bytes, the solver asks CUDA for them, overflow -> global/L2).
void choose_layout(const go_problem* p, int TS, int E_req, int* layout, int* E_out) {
  const int n = p->n;
  const size_t optin = (size_t)p->dev.smem_optin;
  const int cap = p->ops.empty() ? 512 : tsp_jit_cap(TS);
  const int Emax = std::max(1, std::min(8, cap / TS));
  const int E0 = E_req > 0 ? std::min(E_req, Emax) : std::min(4, Emax);
  const int full = p->elem * 2, tri = p->elem * 2 + 1;
  for (int E = E0; E >= 1; --E) {
    if (cta_smem(full, n, E, TS, p->full_bytes) <= optin) { *layout = full; *E_out = E; return; }
    if (n >= 2 && cta_smem(tri, n, E, TS, p->tri_bytes) <= optin) { *layout = tri; *E_out = E; return; }
  }
  *layout = global_layout(p->elem);
  *E_out = E0;
}

// ---- solution layout at the ABI (genes[m][d1*d2] + sizes[m][d1]) <-> device rows --
static void to_device_rows(const go_problem* p, const int32_t* genes, const int32_t* sizes,
                           int m, short* out) {
  if (p->family == 1 && p->row_kind == go::RK_PART) {
    std::fill(out, out + (size_t)m * p->n, (short)0);
    for (int s = 0; s < m; ++s) {
      short* o = out + (size_t)s * p->n;
      int at = 0;
      for (int r = 0; r < p->d1; ++r) {
        const int len = sizes ? sizes[(size_t)s * p->d1 + r] : 0;
        for (int q = 0; q < len && at < p->n_cells; ++q)
          o[at++] = (short)genes[(size_t)s * p->d1 * p->d2 + (size_t)r * p->d2 + q];
        o[p->n_cells + r] = (short)len;
      }
    }
    return;
  }
  for (size_t i = 0; i < (size_t)m * p->n; ++i) out[i] = (short)genes[i];
}

void to_device_rows(const go_problem* p, const int32_t* genes, const int32_t* sizes, int m,
                    std::vector<short>& out) {
  out.assign((size_t)m * p->n, 0);
  to_device_rows(p, genes, sizes, m, out.data());
}

void from_device_rows(const go_problem* p, const short* rows, int m, int32_t* genes,
                      int32_t* sizes) {
  if (p->family == 1 && p->row_kind == go::RK_PART) {
    for (int s = 0; s < m; ++s) {
      const short* o = rows + (size_t)s * p->n;
      int at = 0;
      for (int r = 0; r < p->d1; ++r) {
        const int len = o[p->n_cells + r];
        if (sizes) sizes[(size_t)s * p->d1 + r] = len;
        for (int q = 0; q < p->d2; ++q)
          if (genes) genes[(size_t)s * p->d1 * p->d2 + (size_t)r * p->d2 + q] = q < len ? o[at + q] : 0;
        at += len;
      }
    }
    return;
  }
  const int d1 = p->mf ? p->d1 : 1;  // MULTI_FIXED: every row full
  for (int s = 0; s < m; ++s) {
    if (genes)
      for (int q = 0; q < p->n; ++q) genes[(size_t)s * p->n + q] = rows[(size_t)s * p->n + q];
    if (sizes)
      for (int r = 0; r < d1; ++r) sizes[(size_t)s * d1 + r] = p->n / d1;
  }
}

go::RowArgs row_args(const go_problem* p) {
  go::RowArgs x{};
  x.off1 = p->off1;
  x.off2 = p->off2;
  x.off3 = p->off3;
  x.off4 = p->off4;
  x.capacity = p->capacity;
  x.n_jobs = p->n_jobs;
  x.per_job = p->per_job;
  x.n_mach = p->n_mach;
  // ProblemConfig.n (lns_scope): permutation rows hold n values each (core.py:28-35)
  x.n_cfg = p->row_kind == go::RK_PART ? p->n_cells : (p->mf == 1 ? p->d2 : p->n);
  x.lb = p->lb;
  x.ub = p->ub;
  x.scratch_ints = p->scratch_ints;
  x.n_cells = p->n_cells;
  x.d1 = p->d1;
  x.d2 = p->d2;
  x.tw = p->tw;
  x.obj_weight = 1.0;
  x.enc = p->enc;
  x.okind0 = p->okind0;
  x.okind1 = p->okind1;
  x.mo.m = p->n_obj;
  x.pvar = p->pvar;
  x.mf = p->mf;
  return x;
}

// Scoped device allocations (freed on every return path).
struct DevBufs {
  std::vector<void*> v;
  ~DevBufs() { for (void* q : v) cudaFree(q); }
  template <class T> cudaError_t get(T** q, size_t bytes) {
    cudaError_t e = cudaMalloc((void**)q, std::max<size_t>(bytes, 16));
    if (e == cudaSuccess) v.push_back(*q);
    return e;
  }
};

// Objectives [m][n_obj] and penalties [m] of m device rows (p->n shorts each,
// the layout to_device_rows produces), on the legacy stream.
int eval_device_rows(go_problem* p, const short* d_g, int m, double* d_o, double* d_p) {
  const int n = p->n;
  CK(cudaMemset(d_p, 0, (size_t)m * 8));
  int nn = n;
  if (p->family == 0) {
    void* fn = p->elem == E_I16 ? (void*)go_eval_tsp_i16
                                : (p->elem == E_I32 ? (void*)go_eval_tsp_i32 : (void*)go_eval_tsp_f64);
    const void* inst = p->d_full;
    void* args[] = {(void*)&inst, &nn, (void*)&d_g, &d_o};
    CK(cudaLaunchKernel(fn, dim3(m), dim3(128), args, 0, 0));
    return GO_OK;
  }
  const void* inst = p->d_img;
  unsigned off1 = p->off1;
  if (p->row_kind == go::RK_QAP) {
    void* fn = p->elem == E_I16 ? (void*)go_eval_qap_i16
                                : (p->elem == E_I32 ? (void*)go_eval_qap_i32 : (void*)go_eval_qap_f64);
    void* args[] = {(void*)&inst, &off1, &nn, (void*)&d_g, &d_o};
    CK(cudaLaunchKernel(fn, dim3(m), dim3(128), args, 0, 0));
  } else if (p->row_kind == go::RK_PART) {
    go::RowArgs x = row_args(p);
    void* args[] = {(void*)&inst, &x, (void*)&d_g, &d_o, &d_p};
    CK(cudaLaunchKernel((void*)go_eval_part, dim3(m), dim3(32), args, 0, 0));
  } else if (p->row_kind == go::RK_KNAP) {
    double cap = p->capacity;
    void* args[] = {(void*)&inst, &off1, &nn, &cap, (void*)&d_g, &d_o, &d_p};
    CK(cudaLaunchKernel((void*)go_eval_knap, dim3(m), dim3(128), args, 0, 0));
  } else if (p->row_kind == go::RK_USER) {
    int mm = m;
    void* args[] = {(void*)&inst, &nn, &mm, (void*)&d_g, &d_o, &d_p};
    CU(gohost::drv()->LaunchKernel(p->user_mod.probe, (unsigned)((m + 127) / 128), 1, 1, 128, 1,
                                   1, 0, nullptr, args, nullptr));
  } else {
    int nj = p->n_jobs, pj = p->per_job, nmach = p->n_mach;
    void* args[] = {(void*)&inst, &off1, &nj, &pj, &nmach, (void*)&d_g, &d_o};
    CK(cudaLaunchKernel((void*)go_eval_jsp, dim3(m), dim3(32), args, (size_t)p->scratch_ints * 4, 0));
  }
  CK(cudaDeviceSynchronize());
  return GO_OK;
}

// ---- row family helpers ----------------------------------------------------------
// layout codes for the row family: 10 = instance and lane rows in shared memory,
// 11 = instance global, 12 = lane rows global, 13 = both global (long rows)
bool row_rows_smem(int layout) { return layout == 10 || layout == 11; }
bool row_inst_smem(int layout) { return layout == 10 || layout == 12; }

void* row_kernel(const go_problem* p, int layout, int TS) {
  if (p->row_kind == go::RK_USER) return nullptr;  // JIT (row_kernel_jit)
  const bool s = row_rows_smem(layout);
  if (TS > go::row_max_threads(p->row_kind)) {  // one team wider than the default bound
    if (p->row_kind == go::RK_KNAP) return s ? (void*)go_evolve_knap_w : (void*)go_evolve_knap_gw;
    if (p->row_kind == go::RK_PART) return s ? (void*)go_evolve_part_w : (void*)go_evolve_part_gw;
    return s ? (void*)go_evolve_jsp_w : (void*)go_evolve_jsp_gw;
  }
  if (p->row_kind == go::RK_QAP) {
    if (p->elem == E_I16) return s ? (void*)go_evolve_qap_i16 : (void*)go_evolve_qap_i16_g;
    if (p->elem == E_I32) return s ? (void*)go_evolve_qap_i32 : (void*)go_evolve_qap_i32_g;
    return s ? (void*)go_evolve_qap_f64 : (void*)go_evolve_qap_f64_g;
  }
  if (p->row_kind == go::RK_KNAP) return s ? (void*)go_evolve_knap : (void*)go_evolve_knap_g;
  if (p->row_kind == go::RK_PART) return s ? (void*)go_evolve_part : (void*)go_evolve_part_g;
  return s ? (void*)go_evolve_jsp : (void*)go_evolve_jsp_g;
}

// template arguments of a built-in row problem's evolve kernel (GO_ROW_KERNEL list)
gohost::RowOpsSrc rowops_src(const go_problem* p, bool rows_global) {
  gohost::RowOpsSrc r;
  r.rows_global = rows_global;
  r.gene_type = "short";
  r.elem_type = "double";
  if (p->row_kind == go::RK_QAP) {
    r.kind = "go::RK_QAP";
    r.elem_type = p->elem == E_I16 ? "short" : (p->elem == E_I32 ? "int" : "double");
  } else if (p->row_kind == go::RK_KNAP) {
    r.kind = "go::RK_KNAP";
    r.gene_type = "unsigned char";
  } else if (p->row_kind == go::RK_JSP) {
    r.kind = "go::RK_JSP";
    r.elem_type = "int";
  } else {
    r.kind = "go::RK_PART";
  }
  return r;
}

// the user problem's (or a built-in row problem's with user operators) evolve
// kernel for a layout (the global-rows module is compiled on first use)
int row_kernel_jit(go_problem* p, int layout, CUfunction* out) {
  *out = nullptr;
  if (p->row_kind != go::RK_USER && p->ops.empty()) return GO_OK;  // static kernels
  if (row_rows_smem(layout)) {
    *out = p->user_mod.evolve;
    return GO_OK;
  }
  if (!p->user_mod_g.mod) {
    std::string log;
    int rc;
    if (p->row_kind == go::RK_USER) {
      gohost::UserProblemSrc up = p->user_src;
      up.ops = p->ops;
      up.rows_global = true;
      rc = gohost::jit_build_user(up, &p->user_mod_g, &log);
    } else {
      rc = gohost::jit_build_rowops(rowops_src(p, true), p->ops, &p->user_mod_g, &log);
    }
    if (rc) return fail(rc, "NVRTC build (global lane rows) failed: " + log.substr(0, 2000));
  }
  *out = p->user_mod_g.evolve;
  return GO_OK;
}

unsigned row_team_bytes(const go_problem* p, int TS, int layout = 10) {
  return go::RowSmem::team_bytes(p->n, p->gsize, TS, p->scratch_ints * 4, row_rows_smem(layout));
}

// Layouts 10..13: lane rows / instance in shared memory (10), rows only (11),
// instance only (12), neither (13); the first that fits one team is the
// default.  Lane rows move to global memory (L2-resident, layout 12/13) when
// shared memory would hold fewer than half the teams per SM the thread bound
// allows: C5b's 1000-gene rows take 128 KB per team in shared memory (one
// team per SM, P = 148) against three teams per SM with global rows (P = 444,
// 1.75x the move evaluations per second, tools/row_layout_probe.py).
bool choose_row(const go_problem* p, int TS, int E_req, int* layout, int* E_out, size_t* smem) {
  const size_t optin = (size_t)p->dev.smem_optin;
  const int Emax = std::max(1, std::min(8, go::row_max_threads(p->row_kind) / TS));
  const int E0 = E_req > 0 ? std::min(E_req, Emax) : std::min(4, Emax);
  auto fit = [&](int L, int& E, size_t& need) -> bool {
    const unsigned inst = row_inst_smem(L) ? pad16(p->img_bytes) : 0u;
    const unsigned tb = row_team_bytes(p, TS, L);
    for (E = E0; E >= 1; --E) {
      need = go::PermSmem::team_off(inst) + (size_t)E * tb;
      if (need <= optin) return true;
    }
    return false;
  };
  // teams per SM: E per CTA x CTAs that fit the SM's shared memory (the
  // opt-in limit + the 1 KB per-CTA reserve), at most the thread bound
  auto teams = [&](int E, size_t need) -> int {
    const size_t per_sm = optin + 1024;
    return std::min(E0, E * (int)(per_sm / (need + 1024)));
  };
  int L0 = 10;
  const char* f = getenv("GO_ROW_LAYOUT");  // diagnostic: first layout to try
  if (f) L0 = std::max(10, std::min(13, atoi(f)));
  for (int L = L0; L <= 13; ++L) {
    int E = 0;
    size_t need = 0;
    if (!fit(L, E, need)) continue;
    if (!f && row_rows_smem(L)) {
      for (int Lg = 12; Lg <= 13; ++Lg) {
        int Eg = 0;
        size_t ng = 0;
        if (!fit(Lg, Eg, ng)) continue;
        if (teams(Eg, ng) >= 2 * teams(E, need)) {
          L = Lg;
          E = Eg;
          need = ng;
        }
        break;
      }
    }
    *layout = L;
    *E_out = E;
    *smem = need;
    return true;
  }
  return false;
}

bool seq_supported(const go_problem* p, int id) {
  if (p->family == 0)
    return id == go::SEQ_SWAP || id == go::SEQ_INSERT || id == go::SEQ_REVERSE ||
           id == go::SEQ_OR_OPT || id == go::SEQ_THREE_OPT || id == go::SEQ_OX ||
           id == go::SEQ_SEG_SHUFFLE || id == go::SEQ_SCATTER_SHUFFLE ||
           id == go::SEQ_GUIDED_REBUILD;
  if (id == go::SEQ_SEG_SHUFFLE || id == go::SEQ_SCATTER_SHUFFLE || id == go::SEQ_GUIDED_REBUILD)
    return true;
  if (p->row_kind == go::RK_QAP)
    return id == go::SEQ_SWAP || id == go::SEQ_INSERT || id == go::SEQ_REVERSE ||
           id == go::SEQ_OR_OPT || id == go::SEQ_THREE_OPT || id == go::SEQ_OX;
  if (p->row_kind == go::RK_KNAP)
    return id == go::SEQ_FLIP || id == go::SEQ_SEG_FLIP || id == go::SEQ_UNIFORM_X;
  if (p->row_kind == go::RK_USER) {  // sequence_applicable (operators.py:597-615)
    if (p->enc == go::ENC_PERM)
      return id == go::SEQ_SWAP || id == go::SEQ_INSERT || id == go::SEQ_REVERSE ||
             id == go::SEQ_OR_OPT || id == go::SEQ_THREE_OPT || id == go::SEQ_OX;
    if (p->enc == go::ENC_BINARY)
      return id == go::SEQ_FLIP || id == go::SEQ_SEG_FLIP || id == go::SEQ_UNIFORM_X;
    return id == go::SEQ_RANDOM_RESET || id == go::SEQ_SEG_RESET || id == go::SEQ_UNIFORM_X;
  }
  if (p->row_kind == go::RK_PART)
    return id == go::SEQ_SWAP || id == go::SEQ_INSERT || id == go::SEQ_REVERSE ||
           id == go::SEQ_OR_OPT || id == go::SEQ_THREE_OPT || id == go::SEQ_ROW_SWAP ||
           id == go::SEQ_ROW_SPLIT || id == go::SEQ_ROW_MERGE || id == go::SEQ_OX;
  return id == go::SEQ_RANDOM_RESET || id == go::SEQ_SEG_RESET || id == go::SEQ_UNIFORM_X;
}

int launch_static_or_jit(void* fn, CUfunction jf, dim3 grid, dim3 block, size_t smem,
                         cudaStream_t st, void** args, bool coop = false) {
  if (coop) {  // all CTAs co-resident (grid barrier inside the kernel)
    if (jf) {
      CU(gohost::drv()->LaunchCooperativeKernel(jf, grid.x, grid.y, grid.z, block.x, block.y,
                                                block.z, (unsigned)smem, (CUstream)st, args));
    } else {
      CK(cudaLaunchCooperativeKernel(fn, grid, block, args, smem, st));
    }
    return GO_OK;
  }
  if (jf) {
    CU(gohost::drv()->LaunchKernel(jf, grid.x, grid.y, grid.z, block.x, block.y, block.z, (unsigned)smem,
                      (CUstream)st, args, nullptr));
  } else {
    CK(cudaLaunchKernel(fn, grid, block, args, smem, st));
  }
  return GO_OK;
}

int set_smem_attr(void* fn, CUfunction jf, size_t smem) {
  if (jf) {
    CU(gohost::drv()->FuncSetAttribute(jf, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, (int)smem));
  } else {
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  return GO_OK;
}

// JIT TSP module for a layout and a CTA thread cap (launch bound)
int ensure_jit(go_problem* p, int layout, gohost::JitModule** out, int cap = 0) {
  if (cap <= 0) cap = gohost::jit_max_threads();
  const int key = layout * 4096 + cap;
  auto it = p->jit.find(key);
  if (it != p->jit.end()) {
    *out = &it->second;
    return GO_OK;
  }
  gohost::JitModule m;
  std::string log;
  const int rc = gohost::jit_build_tsp(kLayouts[layout].dist_type, p->ops, &m, &log, cap);
  if (rc) return fail(rc, "NVRTC build failed: " + log);
  p->jit[key] = m;
  *out = &p->jit[key];
  return GO_OK;
}

const void* inst_ptr(const go_problem* p, int layout) {
  return kLayouts[layout].tri ? p->d_tri : p->d_full;
}

size_t inst_img_bytes(const go_problem* p, int layout) {
  return kLayouts[layout].tri ? p->tri_bytes : p->full_bytes;
}

}  // namespace

extern "C" {

int go_problem_layout(const go_problem* p, int64_t* smem_bytes, int32_t* layout) {
  if (!p) return fail(GO_E_INVALID, "null problem");
  int L = 0, E = 0;
  choose_layout(p, 128, 0, &L, &E);
  if (layout) *layout = L;
  if (smem_bytes) *smem_bytes = kLayouts[L].global ? 0 : (int64_t)pad16(inst_img_bytes(p, L));
  return GO_OK;
}

int go_problem_occupancy(go_problem* p, int team_size, int teams_per_cta, int32_t* layout,
                         int32_t* teams_cta, int32_t* teams_per_sm, int64_t* smem_bytes) {
  if (!p || team_size < 1 || team_size > 512) return fail(GO_E_INVALID, "bad arguments");
  CK(cudaSetDevice(p->device));
  const int TS = (team_size + 31) / 32 * 32;
  if (p->family == 1) {
    int L = 0, E = 0;
    size_t smem = 0;
    if (!choose_row(p, TS, teams_per_cta, &L, &E, &smem))
      return fail(GO_E_UNSUPPORTED, "row problem does not fit one team in shared memory");
    void* fn = row_kernel(p, L, TS);
    CUfunction jf = nullptr;
    int jrc = row_kernel_jit(p, L, &jf);
    if (jrc) return jrc;
    int rc = set_smem_attr(fn, jf, smem);
    if (rc) return rc;
    int blocks = 0;
    if (jf) {
      CU(gohost::drv()->OccupancyMaxActiveBlocksPerMultiprocessor(&blocks, jf, E * TS, smem));
    } else {
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, E * TS, smem));
    }
    if (layout) *layout = L;
    if (teams_cta) *teams_cta = E;
    if (teams_per_sm) *teams_per_sm = blocks * E;
    if (smem_bytes) *smem_bytes = (int64_t)smem;
    return GO_OK;
  }
  int L = 0, E = 0;
  choose_layout(p, TS, teams_per_cta, &L, &E);
  const size_t smem = cta_smem(L, p->n, E, TS, inst_img_bytes(p, L));
  CK(cudaFuncSetAttribute(kLayouts[L].evolve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)smem));
  int blocks = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kLayouts[L].evolve, E * TS, smem));
  if (layout) *layout = L;
  if (teams_cta) *teams_cta = E;
  if (teams_per_sm) *teams_per_sm = blocks * E;
  if (smem_bytes) *smem_bytes = (int64_t)smem;
  return GO_OK;
}

int go_eval_batch(go_problem* p, const int32_t* genes, const int32_t* sizes, int m,
                  double* obj_out, double* pen_out) {
  if (!p || !genes || !obj_out || m < 0) return fail(GO_E_INVALID, "bad arguments");
  if (m == 0) return GO_OK;
  CK(cudaSetDevice(p->device));
  std::vector<short> h;
  to_device_rows(p, genes, sizes, m, h);
  short* d_g = nullptr;
  double *d_o = nullptr, *d_p = nullptr;
  CK(cudaMalloc(&d_g, h.size() * 2));
  CK(cudaMalloc(&d_o, (size_t)m * p->n_obj * 8));
  CK(cudaMalloc(&d_p, (size_t)m * 8));
  CK(cudaMemcpy(d_g, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
  const int rc = eval_device_rows(p, d_g, m, d_o, d_p);
  if (rc == GO_OK) {
    CK(cudaMemcpy(obj_out, d_o, (size_t)m * p->n_obj * 8, cudaMemcpyDeviceToHost));
    if (pen_out) CK(cudaMemcpy(pen_out, d_p, (size_t)m * 8, cudaMemcpyDeviceToHost));
  }
  cudaFree(d_g);
  cudaFree(d_o);
  cudaFree(d_p);
  return rc;
}

int go_init_population(go_problem* p, int count, uint64_t seed, uint64_t salt,
                       const int32_t* extra_genes, const int32_t* extra_sizes, int n_extra,
                       int keep, int maximize, double obj_weight, int32_t* genes_out,
                       int32_t* sizes_out, double* obj_out, double* pen_out,
                       int32_t* index_out) {
  if (!p || count < 0 || n_extra < 0 || (n_extra > 0 && !extra_genes)) return fail(GO_E_INVALID, "bad arguments");
  const int M = count + n_extra;
  if (M == 0 || keep < 0 || keep > M) return fail(GO_E_INVALID, "need 0 <= keep <= count + n_extra, pool > 0");
  if (keep > 0 && p->n_obj != 1)
    return fail(GO_E_INVALID, "device selection is single-objective (select fronts on the host)");
  if (!genes_out || !obj_out || !pen_out) return fail(GO_E_INVALID, "null output");
  CK(cudaSetDevice(p->device));
  go::InitArgs a{};
  a.count = count;
  a.W = p->n;
  a.seed = seed;
  a.salt = salt;
  if (p->family == 0 || p->row_kind == go::RK_QAP || (p->row_kind == go::RK_USER && p->enc == 0)) {
    a.kind = 0;  // d1 rows, each a shuffle of range(d2) (engine.py:262-266)
    a.nrows = p->mf ? p->d1 : 1;
    a.n = p->n / a.nrows;
  } else if (p->row_kind == go::RK_PART) {
    a.kind = 1;
    a.n = p->n_cells;
    a.d1 = p->d1;
    a.d2 = p->d2;
  } else {
    a.kind = 2;
    a.n = p->n;
    a.lo = p->lb;
    a.hi = p->ub;
  }
  const int W = p->n, out_n = keep > 0 ? keep : M;
  DevBufs B;
  short *rows = nullptr, *out_rows = nullptr;
  double *d_o = nullptr, *d_p = nullptr;
  int* d_idx = nullptr;
  CK(B.get(&rows, (size_t)M * W * 2));
  CK(B.get(&d_o, (size_t)M * p->n_obj * 8));
  CK(B.get(&d_p, (size_t)M * 8));
  if (a.kind == 1) CK(B.get(&a.scratch, (size_t)count * (2 * a.n + a.d1) * 2));
  a.rows = rows;
  if (count > 0) {
    go::init_random_kernel<<<(count + 127) / 128, 128>>>(a);
    CK(cudaGetLastError());
  }
  if (n_extra > 0) {
    std::vector<short> h;
    to_device_rows(p, extra_genes, extra_sizes, n_extra, h);
    CK(cudaMemcpy(rows + (size_t)count * W, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
  }
  const int rc = eval_device_rows(p, rows, M, d_o, d_p);
  if (rc != GO_OK) return rc;
  std::vector<double> ho((size_t)M * p->n_obj), hp(M);
  CK(cudaMemcpy(ho.data(), d_o, ho.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hp.data(), d_p, hp.size() * 8, cudaMemcpyDeviceToHost));
  std::vector<int> idx(out_n);
  const short* src = rows;
  if (keep > 0) {
    CK(B.get(&out_rows, (size_t)keep * W * 2));
    CK(B.get(&d_idx, (size_t)keep * 4));
    go::SelectArgs s{};
    s.obj = d_o;
    s.pen = d_p;
    s.rows = rows;
    s.M = M;
    s.m_obj = p->n_obj;
    s.W = W;
    s.keep = keep;
    s.w = obj_weight;
    s.maximize = maximize;
    s.out_rows = out_rows;
    s.out_idx = d_idx;
    go::init_select_kernel<<<(M + 255) / 256, 256>>>(s);
    CK(cudaGetLastError());
    CK(cudaMemcpy(idx.data(), d_idx, (size_t)keep * 4, cudaMemcpyDeviceToHost));
    src = out_rows;
  } else {
    for (int i = 0; i < M; ++i) idx[i] = i;
  }
  std::vector<short> hr((size_t)out_n * W);
  CK(cudaMemcpy(hr.data(), src, hr.size() * 2, cudaMemcpyDeviceToHost));
  from_device_rows(p, hr.data(), out_n, genes_out, sizes_out);
  for (int k = 0; k < out_n; ++k) {
    for (int j = 0; j < p->n_obj; ++j) obj_out[(size_t)k * p->n_obj + j] = ho[(size_t)idx[k] * p->n_obj + j];
    pen_out[k] = hp[idx[k]];
    if (index_out) index_out[k] = idx[k];
  }
  return GO_OK;
}

int go_delta_batch(go_problem* p, const int32_t* genes, const int32_t* sizes, int m,
                   const go_move* moves, double penalty_weight, double* delta_out,
                   int32_t* cand_out) {
  (void)sizes;
  (void)penalty_weight;
  if (!p || !genes || !moves || !delta_out || m < 0) return fail(GO_E_INVALID, "bad arguments");
  if (m == 0) return GO_OK;
  CK(cudaSetDevice(p->device));
  const int n = p->n;
  for (int i = 0; i < m * go::MAX_CHAIN; ++i) {
    const go_move& mv = moves[i];
    bool ok = true;
    if (mv.kind == GO_MOVE_SWAP) ok = mv.a >= 0 && mv.b >= 0 && mv.a < n && mv.b < n && mv.a != mv.b;
    else if (mv.kind == GO_MOVE_REVERSE) ok = mv.a >= 0 && mv.a < mv.b && mv.b < n;
    else if (mv.kind == GO_MOVE_SEGMENT)
      ok = mv.b >= 1 && mv.a >= 0 && mv.a + mv.b <= n && mv.c >= 0 && mv.c <= n - mv.b;
    else if (mv.kind >= GO_MOVE_THREE_OPT && mv.kind < GO_MOVE_THREE_OPT + 7)
      ok = 0 < mv.a && mv.a < mv.b && mv.b < mv.c && mv.c < n;
    else ok = mv.kind == GO_MOVE_NONE;
    if (!ok) return fail(GO_E_INVALID, "malformed move at index " + std::to_string(i));
  }
  std::vector<short> h((size_t)m * n);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (short)genes[i];
  short *d_g = nullptr, *d_c = nullptr;
  int* d_m = nullptr;
  double* d_d = nullptr;
  CK(cudaMalloc(&d_g, h.size() * 2));
  CK(cudaMalloc(&d_c, h.size() * 2));
  CK(cudaMalloc(&d_m, (size_t)m * go::MAX_CHAIN * sizeof(go_move)));
  CK(cudaMalloc(&d_d, (size_t)m * 8));
  CK(cudaMemcpy(d_g, h.data(), h.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_m, moves, (size_t)m * go::MAX_CHAIN * sizeof(go_move), cudaMemcpyHostToDevice));
  void* fn = p->elem == E_I16 ? (void*)go_delta_tsp_i16
                              : (p->elem == E_I32 ? (void*)go_delta_tsp_i32 : (void*)go_delta_tsp_f64);
  const void* inst = p->d_full;
  int nn = n;
  void* args[] = {(void*)&inst, &nn, &d_g, &d_m, &d_d, &d_c};
  CK(cudaLaunchKernel(fn, dim3(m), dim3(128), args, pad16((size_t)n * 2), 0));
  CK(cudaMemcpy(delta_out, d_d, (size_t)m * 8, cudaMemcpyDeviceToHost));
  if (cand_out) {
    CK(cudaMemcpy(h.data(), d_c, h.size() * 2, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < h.size(); ++i) cand_out[i] = h[i];
  }
  cudaFree(d_g);
  cudaFree(d_c);
  cudaFree(d_m);
  cudaFree(d_d);
  return GO_OK;
}

int go_jit_compile(int layout, const go_custom_op* ops, int n_ops, char* log, int log_len,
                   char* key_hex65) {
  if (layout < 0 || layout > 8 || n_ops < 0 || (n_ops && !ops)) return fail(GO_E_INVALID, "bad arguments");
  std::vector<gohost::UserOpSrc> v;
  for (int i = 0; i < n_ops; ++i)
    v.push_back({ops[i].id, ops[i].name ? ops[i].name : "op", ops[i].cuda_body ? ops[i].cuda_body : ""});
  std::string cubin, key, lg;
  bool hit = false;
  const int rc = gohost::jit_compile_tsp(kLayouts[layout].dist_type, v, &cubin, &key, &hit, &lg);
  if (log && log_len > 0) snprintf(log, log_len, "%s", lg.c_str());
  if (key_hex65) snprintf(key_hex65, 65, "%s", key.c_str());
  if (rc) return fail(rc, "NVRTC: " + lg.substr(0, 2000));
  return GO_OK;
}

}  // extern "C"

// register_custom (operators.py:634-669) for a user problem: each operator is
// compiled into the problem's NVRTC module on its own (a compile error excludes
// only it), probed once on the probe solution (a device error or an invalid
// result excludes it), and the kept ones are built into the problem's module.
template <class Note>
static int set_user_problem_ops(go_problem* p, const go_custom_op* ops, int n_ops,
                                const int32_t* probe_genes, uint64_t probe_seed,
                                int32_t* status_out, Note note) {
  std::vector<gohost::UserOpSrc> keep;
  const int n = p->n;
  for (int i = 0; i < n_ops; ++i) {
    status_out[i] = 0;
    if (ops[i].id < 100) return fail(GO_E_INVALID, "custom operator id must be >= 100");
    if (!ops[i].cuda_body) {
      note(i, "no CUDA snippet");
      continue;
    }
    gohost::UserOpSrc s{ops[i].id, ops[i].name ? ops[i].name : "op", ops[i].cuda_body};
    gohost::UserProblemSrc up = p->user_src;
    up.ops = {s};
    gohost::JitModule m;
    std::string log;
    if (gohost::jit_build_user(up, &m, &log)) {
      note(i, "compile failed: " + log.substr(0, 400));
      continue;
    }
    std::vector<short> h(n);
    for (int j = 0; j < n; ++j) h[j] = (short)probe_genes[j];
    DevBufs B;
    short* d_g = nullptr;
    int* d_e = nullptr;
    CK(B.get(&d_g, (size_t)n * 2));
    CK(B.get(&d_e, sizeof(int)));
    CK(cudaMemcpy(d_g, h.data(), (size_t)n * 2, cudaMemcpyHostToDevice));
    CK(cudaMemset(d_e, 0, sizeof(int)));
    auto mix = [](uint64_t hh, uint64_t part) {
      hh ^= part;
      hh *= 0xBF58476D1CE4E5B9ull;
      hh ^= hh >> 27;
      hh *= 0x94D049BB133111EBull;
      hh ^= hh >> 31;
      return hh;
    };
    unsigned long long key =
        mix(mix(mix(0x9E3779B97F4A7C15ull, probe_seed), 4), (uint64_t)ops[i].id);
    go::RowArgs x = row_args(p);
    const void* inst = p->d_img;
    int nn = n, slot = 0;
    void* args[] = {(void*)&inst, &x, &nn, &slot, &key, &d_g, &d_e};
    CU(gohost::drv()->LaunchKernel(m.probe_op, 1, 1, 1, 32, 1, 1, 0, 0, args, nullptr));
    const cudaError_t ce = cudaDeviceSynchronize();
    gohost::drv()->ModuleUnload(m.mod);
    if (ce != cudaSuccess) return fail(GO_E_CUDA, std::string("probe kernel: ") + cudaGetErrorString(ce));
    int err = 0;
    CK(cudaMemcpy(&err, d_e, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h.data(), d_g, (size_t)n * 2, cudaMemcpyDeviceToHost));
    bool valid = err == 0;
    if (p->enc == go::ENC_PERM) {  // every row a permutation of 0 .. d2-1
      for (int r = 0; r < p->d1 && valid; ++r) {
        std::vector<char> seen(p->d2, 0);
        for (int j = 0; j < p->d2 && valid; ++j) {
          const int v = h[(size_t)r * p->d2 + j];
          if (v < 0 || v >= p->d2 || seen[v]) valid = false;
          else seen[v] = 1;
        }
      }
    } else {
      for (int j = 0; j < n && valid; ++j) valid = h[j] >= p->lb && h[j] <= p->ub;
    }
    if (!valid) {
      note(i, err ? "probe raised a device error" : "probe output invalid");
      continue;
    }
    keep.push_back(s);
    status_out[i] = 1;
    note(i, "registered");
  }
  gohost::UserProblemSrc up = p->user_src;
  up.ops = keep;
  gohost::JitModule m;
  std::string log;
  const int rc = gohost::jit_build_user(up, &m, &log);
  if (rc) return fail(rc, "NVRTC build of the user problem with its operators failed: " + log.substr(0, 2000));
  if (p->user_mod.mod && gohost::drv()) gohost::drv()->ModuleUnload(p->user_mod.mod);
  if (p->user_mod_g.mod && gohost::drv()) gohost::drv()->ModuleUnload(p->user_mod_g.mod);
  p->user_mod_g = gohost::JitModule{};
  p->user_mod = m;
  p->ops = keep;
  return GO_OK;
}

// register_custom (operators.py:634-669) for a BUILT-IN row problem (QAP,
// knapsack, JSP-int, VRPTW / CVRP and the routing variants): each operator is
// compiled alone into the problem's hand-written evolve kernel (a compile
// error excludes only it), probed once on the probe solution (device error
// or an invalid result excludes it), then the kept ones are built together.
template <class Note>
static int set_rowops_problem_ops(go_problem* p, const go_custom_op* ops, int n_ops,
                                  const int32_t* probe_genes, const int32_t* probe_sizes,
                                  uint64_t probe_seed, int32_t* status_out, Note note) {
  std::vector<gohost::UserOpSrc> keep;
  const int n = p->n;  // device row length (partitions: cells + route sizes)
  std::vector<short> h0;
  to_device_rows(p, probe_genes, probe_sizes, 1, h0);
  auto valid_row = [&](const std::vector<short>& h) {
    if (p->row_kind == go::RK_PART) {
      int tot = 0;
      for (int r = 0; r < p->d1; ++r) {
        const int sz = h[p->n_cells + r];
        if (sz < 0 || sz > p->d2) return false;
        tot += sz;
      }
      if (tot != p->n_cells) return false;
      std::vector<char> seen(p->n_cells, 0);
      for (int q = 0; q < p->n_cells; ++q) {
        const int v = h[q];
        if (v < 0 || v >= p->n_cells || seen[v]) return false;
        seen[v] = 1;
      }
      return true;
    }
    if (p->row_kind == go::RK_QAP) {
      std::vector<char> seen(n, 0);
      for (int j = 0; j < n; ++j) {
        if (h[j] < 0 || h[j] >= n || seen[h[j]]) return false;
        seen[h[j]] = 1;
      }
      return true;
    }
    const int lo = p->row_kind == go::RK_KNAP ? 0 : p->lb;
    const int hi = p->row_kind == go::RK_KNAP ? 1 : p->ub;
    for (int j = 0; j < n; ++j)
      if (h[j] < lo || h[j] > hi) return false;
    return true;
  };
  auto mix = [](uint64_t hh, uint64_t part) {
    hh ^= part;
    hh *= 0xBF58476D1CE4E5B9ull;
    hh ^= hh >> 27;
    hh *= 0x94D049BB133111EBull;
    hh ^= hh >> 31;
    return hh;
  };
  for (int i = 0; i < n_ops; ++i) {
    status_out[i] = 0;
    if (ops[i].id < 100) return fail(GO_E_INVALID, "custom operator id must be >= 100");
    if (!ops[i].cuda_body) {
      note(i, "no CUDA snippet");
      continue;
    }
    gohost::UserOpSrc src{ops[i].id, ops[i].name ? ops[i].name : "op", ops[i].cuda_body};
    gohost::JitModule m;
    std::string log;
    if (gohost::jit_build_rowops(rowops_src(p, false), {src}, &m, &log)) {
      note(i, "compile failed: " + log.substr(0, 400));
      continue;
    }
    std::vector<short> h = h0;
    DevBufs B;
    short* d_g = nullptr;
    int* d_e = nullptr;
    CK(B.get(&d_g, (size_t)n * 2));
    CK(B.get(&d_e, sizeof(int)));
    CK(cudaMemcpy(d_g, h.data(), (size_t)n * 2, cudaMemcpyHostToDevice));
    CK(cudaMemset(d_e, 0, sizeof(int)));
    unsigned long long key =
        mix(mix(mix(0x9E3779B97F4A7C15ull, probe_seed), 4), (uint64_t)ops[i].id);
    go::RowArgs x = row_args(p);
    const void* inst = p->d_img;
    int nn = p->row_kind == go::RK_PART ? p->n_cells : n, slot = 0;
    void* args[] = {(void*)&inst, &x, &nn, &slot, &key, &d_g, &d_e};
    CU(gohost::drv()->LaunchKernel(m.probe_op, 1, 1, 1, 32, 1, 1, 0, 0, args, nullptr));
    const cudaError_t ce = cudaDeviceSynchronize();
    gohost::drv()->ModuleUnload(m.mod);
    if (ce != cudaSuccess) return fail(GO_E_CUDA, std::string("probe kernel: ") + cudaGetErrorString(ce));
    int err = 0;
    CK(cudaMemcpy(&err, d_e, sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h.data(), d_g, (size_t)n * 2, cudaMemcpyDeviceToHost));
    if (err || !valid_row(h)) {
      note(i, err ? "probe raised a device error" : "probe output invalid");
      continue;
    }
    keep.push_back(src);
    status_out[i] = 1;
    note(i, "registered");
  }
  if (p->user_mod.mod && gohost::drv()) gohost::drv()->ModuleUnload(p->user_mod.mod);
  if (p->user_mod_g.mod && gohost::drv()) gohost::drv()->ModuleUnload(p->user_mod_g.mod);
  p->user_mod = gohost::JitModule{};
  p->user_mod_g = gohost::JitModule{};
  p->ops = keep;
  if (keep.empty()) return GO_OK;  // the static kernels again
  gohost::JitModule m;
  std::string log;
  const int rc = gohost::jit_build_rowops(rowops_src(p, false), keep, &m, &log);
  if (rc) return fail(rc, "NVRTC build of the row kernel with its operators failed: " + log.substr(0, 2000));
  p->user_mod = m;
  return GO_OK;
}

extern "C" {

int go_problem_set_custom_ops(go_problem* p, const go_custom_op* ops, int n_ops,
                              const int32_t* probe_genes, const int32_t* probe_sizes,
                              uint64_t probe_seed, int32_t* status_out, char* msg_out,
                              int msg_len) {
  if (!p || (n_ops > 0 && !ops) || !status_out) return fail(GO_E_INVALID, "bad arguments");
  CK(cudaSetDevice(p->device));
  for (auto& kv : p->jit)
    if (kv.second.mod && gohost::drv()) gohost::drv()->ModuleUnload(kv.second.mod);
  p->jit.clear();
  p->ops.clear();
  auto note = [&](int i, const std::string& m) {
    if (msg_out && msg_len > 0) snprintf(msg_out + (size_t)i * msg_len, msg_len, "%s", m.c_str());
  };
  if (p->row_kind == go::RK_USER) return set_user_problem_ops(p, ops, n_ops, probe_genes,
                                                               probe_seed, status_out, note);
  if (p->family == 1) return set_rowops_problem_ops(p, ops, n_ops, probe_genes, probe_sizes,
                                                    probe_seed, status_out, note);
  int layout = 0, E = 0;
  choose_layout(p, 128, 0, &layout, &E);
  // compile each operator on its own first so a broken snippet only excludes
  // itself (operators.py:649-657); then probe it on the device (:658-665)
  std::vector<gohost::UserOpSrc> keep;
  for (int i = 0; i < n_ops; ++i) {
    status_out[i] = 0;
    if (ops[i].id < 100) return fail(GO_E_INVALID, "custom operator id must be >= 100");
    if (!ops[i].cuda_body) {
      note(i, "no CUDA snippet");
      continue;
    }
    gohost::UserOpSrc s{ops[i].id, ops[i].name ? ops[i].name : "op", ops[i].cuda_body};
    gohost::JitModule m;
    std::string log;
    const int rc = gohost::jit_build_tsp(kLayouts[layout].dist_type, {s}, &m, &log);
    if (rc) {
      note(i, "compile failed: " + log.substr(0, 400));
      continue;
    }
    // probe: one application on the probe tour with stream mix64(seed, 4, id)
    const int n = p->n;
    short* d_g = nullptr;
    int* d_e = nullptr;
    std::vector<short> h(n);
    for (int j = 0; j < n; ++j) h[j] = (short)probe_genes[j];
    CK(cudaMalloc(&d_g, (size_t)n * 2));
    CK(cudaMalloc(&d_e, sizeof(int)));
    CK(cudaMemcpy(d_g, h.data(), (size_t)n * 2, cudaMemcpyHostToDevice));
    CK(cudaMemset(d_e, 0, sizeof(int)));
    auto mix = [](uint64_t hh, uint64_t part) {
      hh ^= part;
      hh *= 0xBF58476D1CE4E5B9ull;
      hh ^= hh >> 27;
      hh *= 0x94D049BB133111EBull;
      hh ^= hh >> 31;
      return hh;
    };
    unsigned long long key = mix(mix(mix(0x9E3779B97F4A7C15ull, probe_seed), 4), (uint64_t)ops[i].id);
    const void* inst = inst_ptr(p, layout);
    int nn = n, kind = go::SEQ_CUSTOM_BASE + 0;
    void* args[] = {(void*)&inst, &nn, &kind, &key, &d_g, &d_e};
    CU(gohost::drv()->LaunchKernel(m.probe, 1, 1, 1, 128, 1, 1, pad16((size_t)n * 2), 0, args, nullptr));
    cudaError_t ce = cudaDeviceSynchronize();
    int err = 0;
    if (ce == cudaSuccess) {
      cudaMemcpy(&err, d_e, sizeof(int), cudaMemcpyDeviceToHost);
      cudaMemcpy(h.data(), d_g, (size_t)n * 2, cudaMemcpyDeviceToHost);
    }
    cudaFree(d_g);
    cudaFree(d_e);
    gohost::drv()->ModuleUnload(m.mod);
    if (ce != cudaSuccess) return fail(GO_E_CUDA, std::string("probe kernel: ") + cudaGetErrorString(ce));
    std::vector<char> seen(n, 0);
    bool valid = err == 0;
    for (int j = 0; j < n && valid; ++j) {
      if (h[j] < 0 || h[j] >= n || seen[h[j]]) valid = false;
      else seen[h[j]] = 1;
    }
    if (!valid) {
      note(i, err ? "probe raised a device error (out-of-range access or malformed move)"
                  : "probe output invalid");
      continue;
    }
    keep.push_back(s);
    status_out[i] = 1;
    note(i, "registered");
  }
  p->ops = keep;
  return GO_OK;
}

// ---- engine ---------------------------------------------------------------------
int go_engine_create(go_problem* p, const go_engine_config* c, go_engine** out) {
  if (!p || !c || !out) return fail(GO_E_INVALID, "null argument");
  if (c->population < 1) return fail(GO_E_INVALID, "population must be >= 1");
  if (c->team_size < 1 || c->team_size > 512)
    return fail(GO_E_UNSUPPORTED, "team_size must be in [1, 512] on the device path");
  if (c->aos_interval < 1 || c->elite_interval < 1 || c->migration_interval < 1)
    return fail(GO_E_INVALID, "intervals must be >= 1");
  if (c->islands < 1 || c->islands > 64 || c->islands > c->population)
    return fail(GO_E_INVALID, "islands must be in [1, min(64, population)]");
  if (c->top_n < 1) return fail(GO_E_INVALID, "top_n must be >= 1");
  CK(cudaSetDevice(p->device));
  std::unique_ptr<go_engine> e(new go_engine());
  e->prob = p;
  e->cfg = *c;
  e->obj_sign_over_w = (c->maximize ? -1.0 : 1.0) / (c->obj_weight > 0 ? c->obj_weight : 1.0);
  e->P = c->population;
  e->T = c->team_size;
  e->TS = (c->team_size + 31) / 32 * 32;
  e->n = p->n;
  e->W = p->n;
  if (p->family == 1) {
    if (!choose_row(p, e->TS, c->teams_per_cta, &e->layout, &e->E, &e->smem))
      return fail(GO_E_UNSUPPORTED, "row problem does not fit one team in shared memory");
    e->inst = p->d_img;
    e->inst_bytes = row_inst_smem(e->layout) ? pad16(p->img_bytes) : 0u;
    e->k_evolve = row_kernel(p, e->layout, e->TS);
    if (int jrc = row_kernel_jit(p, e->layout, &e->k_evolve_jit)) return jrc;
  } else {
  choose_layout(p, e->TS, c->teams_per_cta, &e->layout, &e->E);
  const LayoutInfo& L = kLayouts[e->layout];
  e->inst = inst_ptr(p, e->layout);
  e->inst_bytes = L.global ? 0u : pad16(inst_img_bytes(p, e->layout));
  e->smem = cta_smem(e->layout, e->n, e->E, e->TS, inst_img_bytes(p, e->layout));
  }
  e->grid = (e->P + e->E - 1) / e->E;
  if (p->family == 0 && !p->ops.empty()) {
    gohost::JitModule* m = nullptr;
    int rc = ensure_jit(p, e->layout, &m, tsp_jit_cap(e->TS));
    if (rc) return rc;
    e->k_evolve_jit = m->evolve;
  } else if (p->family == 0) {
    e->k_evolve = kLayouts[e->layout].evolve;
  }
  int rc = set_smem_attr(e->k_evolve, e->k_evolve_jit, e->smem);
  if (rc) return rc;
  // resident teams per SM for the population sizing rule (paper §4.4)
  int blocks = 0;
  if (e->k_evolve_jit) {
    CU(gohost::drv()->OccupancyMaxActiveBlocksPerMultiprocessor(&blocks, e->k_evolve_jit, e->E * e->TS, e->smem));
  } else {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, e->k_evolve, e->E * e->TS, e->smem));
  }
  e->teams_per_sm = blocks * e->E;
  if (blocks < 1) return fail(GO_E_UNSUPPORTED, "evolve kernel does not fit on an SM");
  e->coop = (long long)blocks * p->dev.sm >= e->grid;
  e->mo.m = p->n_obj;
  e->mo.lex = c->lex ? 1 : 0;
  e->mo.first = c->lex_first == 1 ? 1 : 0;
  e->mo.maxmask = (c->maximize ? 1 : 0) | (c->maximize2 ? 2 : 0);
  e->mo.tol[0] = c->lex_tol[0];
  e->mo.tol[1] = c->lex_tol[1];
  const bool multi = p->n_obj == 2 || e->mo.lex;
  if (multi && !(p->family == 1 && (p->row_kind == go::RK_PART || p->row_kind == go::RK_USER)))
    return fail(GO_E_UNSUPPORTED,
                "multi-objective / Lexicographic runs: routing and user problems only");
  if (e->mo.first >= e->mo.m) return fail(GO_E_INVALID, "lex_first outside the objectives");

  // per-thread stack: the row kernels' guided rebuild nests numpy's recursive
  // pairwise sum (go_part.cuh) below ~1 KB of frames; the default limit is 1 KB
  size_t stack = 0;
  CK(cudaDeviceGetLimit(&stack, cudaLimitStackSize));
  if (stack < kStackBytes) CK(cudaDeviceSetLimit(cudaLimitStackSize, kStackBytes));
  CK(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking));
  const size_t P = e->P, W = e->W;
  CK(cudaMalloc(&e->genes, P * W * 2));
  CK(cudaMalloc(&e->best_genes, P * W * 2));
  CK(cudaMalloc(&e->gbest_genes, W * 2));
  CK(cudaMalloc(&e->scratch, (size_t)std::max(c->islands, std::min(c->top_n, 64)) * W * 2));
  CK(cudaMalloc(&e->scal, P * 8));
  CK(cudaMalloc(&e->pen, P * 8));
  CK(cudaMalloc(&e->best_scal, P * 8));
  CK(cudaMalloc(&e->best_pen, P * 8));
  CK(cudaMalloc(&e->best_gen, P * 8));
  CK(cudaMalloc(&e->usage, P * go::MAX_SEQ * 4));
  CK(cudaMalloc(&e->impr, P * go::MAX_SEQ * 4));
  CK(cudaMalloc(&e->k_usage, P * 3 * 4));
  CK(cudaMalloc(&e->k_impr, P * 3 * 4));
  CK(cudaMalloc(&e->agg, 70 * 8));
  CK(cudaMemset(e->agg, 0, 70 * 8));
  CK(cudaMalloc(&e->rec_scal, (size_t)go::MAX_CHUNK * P * 8));
  CK(cudaMalloc(&e->rec_pen, (size_t)go::MAX_CHUNK * P * 8));
  CK(cudaMalloc(&e->temps, (size_t)go_engine::kDepth * go::MAX_CHUNK * 8));
  CK(cudaMallocHost(&e->h_temps, (size_t)go_engine::kDepth * go::MAX_CHUNK * 8));
  CK(cudaMalloc(&e->reg, sizeof(go::RegistryDev)));
  CK(cudaMalloc(&e->gs, sizeof(go::GlobalState)));
  if (multi) {
    CK(cudaMalloc(&e->obj2, P * 2 * 8));
    CK(cudaMalloc(&e->best_obj2, P * 2 * 8));
    CK(cudaMalloc(&e->rec_obj2, (size_t)go::MAX_CHUNK * P * 2 * 8));
  }
  CK(cudaHostAlloc(&e->h_stop, sizeof(int), cudaHostAllocMapped));
  *e->h_stop = 0;
  CK(cudaHostGetDevicePointer((void**)&e->d_stop_map, e->h_stop, 0));
  for (auto& ev : e->ring_ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  for (auto& ev : e->k_beg) CK(cudaEventCreate(&ev));
  for (auto& ev : e->k_end) CK(cudaEventCreate(&ev));
  CK(cudaEventCreate(&e->t_start));
  CK(cudaEventCreate(&e->t_stop));
  go::GlobalState gs{};
  gs.gev = -1;
  CK(cudaMemcpy(e->gs, &gs, sizeof(gs), cudaMemcpyHostToDevice));
  *out = e.release();
  return GO_OK;
}

int go_engine_destroy(go_engine* e) {
  if (!e) return GO_OK;
  cudaSetDevice(e->prob->device);
  if (e->stream) cudaStreamSynchronize(e->stream);
  void* bufs[] = {e->genes, e->best_genes, e->gbest_genes, e->scratch, e->scal, e->pen,
                  e->best_scal, e->best_pen, e->best_gen, e->usage, e->impr, e->k_usage,
                  e->k_impr, e->agg, e->rec_scal, e->rec_pen, e->temps, e->reg, e->gs,
                  e->history, e->snap, e->prog, e->lane_rows, e->obj2, e->best_obj2,
                  e->rec_obj2};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (e->h_temps) cudaFreeHost(e->h_temps);
  if (e->h_stop) cudaFreeHost(e->h_stop);
  if (e->h_pin) cudaFreeHost(e->h_pin);
  if (e->pin_ev) cudaEventDestroy(e->pin_ev);
  for (auto& ev : e->ring_ev)
    if (ev) cudaEventDestroy(ev);
  for (int i = 0; i < go_engine::kDepth; ++i) {
    if (e->k_beg[i]) cudaEventDestroy(e->k_beg[i]);
    if (e->k_end[i]) cudaEventDestroy(e->k_end[i]);
  }
  if (e->t_start) cudaEventDestroy(e->t_start);
  if (e->t_stop) cudaEventDestroy(e->t_stop);
  if (e->stream) cudaStreamDestroy(e->stream);
  delete e;
  return GO_OK;
}

int go_engine_set_registry(go_engine* e, int nseq, const int32_t* ids, const double* weights,
                           const double* floors, const double* caps, double total,
                           const double* k_weights) {
  if (!e || nseq < 1 || nseq > 31 || !ids || !weights || !k_weights)
    return fail(GO_E_INVALID, "registry needs 1..31 sequences");
  go::RegistryDev r{};
  r.nseq = nseq;
  double acc = 0.0;
  for (int i = 0; i < nseq; ++i) {
    const int id = ids[i];
    int kind = -1;
    if (id >= 0 && id < 32 && seq_supported(e->prob, id)) {
      kind = id;
    } else if (id >= 100) {
      for (size_t s = 0; s < e->prob->ops.size(); ++s)
        if (e->prob->ops[s].id == id) kind = go::SEQ_CUSTOM_BASE + (int)s;
    }
    if (kind < 0)
      return fail(GO_E_UNSUPPORTED, "sequence id " + std::to_string(id) +
                                        " has no device implementation for this problem");
    if (id >= 100 && !e->k_evolve_jit)
      return fail(GO_E_INVALID, "custom sequence registered after engine creation");
    r.kind[i] = kind;
    r.ids[i] = id;
    r.w[i] = weights[i];
    r.floor_[i] = floors ? floors[i] : 0.0;
    r.cap[i] = caps ? caps[i] : INFINITY;
    acc += weights[i];  // sample_sequence's running sum (aos.py:169-175)
    r.cum[i] = acc;
  }
  r.total = total;
  for (int j = 0; j < 3; ++j) r.kw[j] = k_weights[j];
  e->nseq = nseq;
  CK(cudaSetDevice(e->prob->device));
  e->xover = false;
  for (int i = 0; i < nseq; ++i) e->xover |= ids[i] == go::SEQ_OX || ids[i] == go::SEQ_UNIFORM_X;
  if (e->xover && !e->snap) {
    CK(cudaMalloc(&e->snap, (size_t)go::SNAP_DEPTH * e->P * e->W * 2));
    CK(cudaMalloc(&e->prog, (size_t)e->P * 4));
  }
  bool whole_row = false;
  for (int i = 0; i < nseq; ++i)
    whole_row |= ids[i] == go::SEQ_OX || ids[i] == go::SEQ_SEG_SHUFFLE ||
                 ids[i] == go::SEQ_SCATTER_SHUFFLE || ids[i] == go::SEQ_GUIDED_REBUILD;
  if (e->prob->family == 0 && whole_row && !e->lane_rows)
    CK(cudaMalloc(&e->lane_rows, (size_t)e->P * e->T * 2 * e->n * 2));
  if (e->prob->family == 1 && !row_rows_smem(e->layout) && !e->lane_rows)  // long rows
    CK(cudaMalloc(&e->lane_rows, (size_t)e->P * e->TS *
                                     go::RowSmem::row_stride(e->n, e->prob->gsize)));
  CK(cudaMemcpyAsync(e->reg, &r, sizeof(r), cudaMemcpyHostToDevice, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  return GO_OK;
}

// Pinned staging area of at least `bytes`, free to write (the previous copy
// out of it has completed).
static unsigned char* engine_pinned(go_engine* e, size_t bytes) {
  if (e->pin_ev) {
    if (cudaEventSynchronize(e->pin_ev) != cudaSuccess) return nullptr;
  } else if (cudaEventCreateWithFlags(&e->pin_ev, cudaEventDisableTiming) != cudaSuccess) {
    return nullptr;
  }
  if (bytes > e->h_pin_bytes) {
    if (e->h_pin) cudaFreeHost(e->h_pin);
    e->h_pin = nullptr;
    e->h_pin_bytes = 0;
    if (cudaHostAlloc((void**)&e->h_pin, bytes, cudaHostAllocDefault) != cudaSuccess) return nullptr;
    e->h_pin_bytes = bytes;
  }
  return e->h_pin;
}

static size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

// Replaces the population (engine.py:538-560 semantics: best-evers reset to the
// new rows, the global best re-selected).  The rows and per-evolver values are
// staged once into pinned memory and copied asynchronously on the engine
// stream (duplicates device-to-device); go_engine_run orders after them.
int go_engine_set_population(go_engine* e, const int32_t* genes, const int32_t* sizes,
                             const double* obj, const double* pen) {
  if (!e || !genes || !obj) return fail(GO_E_INVALID, "bad arguments");
  CK(cudaSetDevice(e->prob->device));
  const size_t P = e->P, W = e->W;
  const size_t o_g = 0, o_sc = align16(P * W * 2), o_pe = o_sc + P * 8, o_o2 = o_pe + P * 8,
               o_gs = align16(o_o2 + P * 16), total = o_gs + sizeof(go::GlobalState);
  unsigned char* h = engine_pinned(e, total);
  if (!h) return fail(GO_E_CUDA, "pinned staging allocation failed");
  short* g = (short*)(h + o_g);
  double *sc = (double*)(h + o_sc), *pe = (double*)(h + o_pe), *o2 = (double*)(h + o_o2);
  to_device_rows(e->prob, genes, sizes, (int)P, g);
  const double w = e->cfg.obj_weight > 0 ? e->cfg.obj_weight : 1.0;
  const int m = e->mo.m;
  int best = 0;
  for (size_t i = 0; i < P; ++i) {
    const double o0 = obj[i * m], o1 = m == 2 ? obj[i * m + 1] : 0.0;
    sc[i] = 0.0 + w * (e->cfg.maximize ? -o0 : o0);  // scalarize (core.py:303-307)
    if (m == 2) sc[i] = sc[i] + e->cfg.obj_weight2 * (e->cfg.maximize2 ? -o1 : o1);
    o2[2 * i] = o0;
    o2[2 * i + 1] = o1;
    pe[i] = pen ? pen[i] : 0.0;
  }
  auto cmp = [&](size_t a, size_t b) -> int {  // compare (core.py:315-347)
    const bool fa = pe[a] == 0.0, fb = pe[b] == 0.0;
    if (fa != fb) return fa ? -1 : 1;
    if (!fa && pe[a] != pe[b]) return pe[a] < pe[b] ? -1 : 1;
    if (!e->mo.lex) return sc[a] < sc[b] ? -1 : (sc[b] < sc[a] ? 1 : 0);
    for (int k = 0; k < m; ++k) {
      const int i = k == 0 ? e->mo.first : 1 - e->mo.first;
      const double x = o2[2 * a + i], y = o2[2 * b + i];
      if (std::fabs(x - y) <= e->mo.tol[i]) continue;
      return (x < y) != ((e->mo.maxmask >> i & 1) != 0) ? -1 : 1;  // low wins unless Maximize
    }
    return 0;
  };
  for (size_t i = 1; i < P; ++i)  // _best_index (engine.py:467-472)
    if (cmp(i, (size_t)best) < 0) best = (int)i;
  go::GlobalState* gs = (go::GlobalState*)(h + o_gs);
  *gs = go::GlobalState{};
  gs->gscal = sc[best];
  gs->gpen = pe[best];
  gs->gobj[0] = o2[2 * best];
  gs->gobj[1] = o2[2 * best + 1];
  gs->gev = -1;
  gs->ggen = 0;
  const cudaStream_t s = e->stream;
  const cudaMemcpyKind H2D = cudaMemcpyHostToDevice, D2D = cudaMemcpyDeviceToDevice;
  if (e->obj2) {
    CK(cudaMemcpyAsync(e->obj2, o2, P * 16, H2D, s));
    CK(cudaMemcpyAsync(e->best_obj2, e->obj2, P * 16, D2D, s));
  }
  CK(cudaMemcpyAsync(e->genes, g, P * W * 2, H2D, s));
  CK(cudaMemcpyAsync(e->best_genes, e->genes, P * W * 2, D2D, s));
  CK(cudaMemcpyAsync(e->gbest_genes, e->genes + (size_t)best * W, W * 2, D2D, s));
  CK(cudaMemcpyAsync(e->scal, sc, P * 8, H2D, s));
  CK(cudaMemcpyAsync(e->best_scal, e->scal, P * 8, D2D, s));
  CK(cudaMemcpyAsync(e->pen, pe, P * 8, H2D, s));
  CK(cudaMemcpyAsync(e->best_pen, e->pen, P * 8, D2D, s));
  CK(cudaMemsetAsync(e->best_gen, 0, P * 8, s));
  CK(cudaMemcpyAsync(e->gs, gs, sizeof(*gs), H2D, s));
  CK(cudaMemsetAsync(e->agg, 0, 70 * 8, s));
  CK(cudaEventRecord(e->pin_ev, s));
  *e->h_stop = 0;
  e->gen_enqueued = 0;
  return GO_OK;
}

int go_engine_set_history(go_engine* e, int enabled) {
  if (!e) return fail(GO_E_INVALID, "null engine");
  e->history_on = enabled != 0;
  return GO_OK;
}

// Evolve-kernel arguments of an engine (everything but the chunk: gen0,
// ngen, temps are set per launch).
static void build_evolve_args(go_engine* e, go::EvolveArgs& a, go::RowArgs& x) {
  const go_engine_config& c = e->cfg;
  a = go::EvolveArgs{};
  x = go::RowArgs{};
  a.inst = e->inst;
  a.inst_bytes = e->inst_bytes;
  a.n = e->n;
  a.genes = e->genes;
  a.scal = e->scal;
  a.pen = e->pen;
  a.best_genes = e->best_genes;
  a.best_scal = e->best_scal;
  a.best_pen = e->best_pen;
  a.best_gen = e->best_gen;
  a.has_target = c.has_target;
  a.target = c.target_objective;
  a.obj_sign_over_w = e->obj_sign_over_w;
  a.usage = e->usage;
  a.impr = e->impr;
  a.k_usage = e->k_usage;
  a.k_impr = e->k_impr;
  a.rec_scal = e->rec_scal;
  a.rec_pen = e->rec_pen;
  a.reg = e->reg;
  a.gs = e->gs;
  a.seed = c.seed;
  a.P = e->P;
  a.T = e->T;
  a.E = e->E;
  a.ev_offset = c.evolver_offset;
  a.team_stride = e->TS;
  a.snap = e->xover ? e->snap : nullptr;
  a.obj2 = e->obj2;
  a.best_obj2 = e->best_obj2;
  a.rec_obj2 = e->rec_obj2;
  a.lane_rows = e->lane_rows;
  a.prog = e->prog;
  a.islands = c.islands;
  if (e->prob->family == 1) {
    const go_problem* p = e->prob;
    a.team_smem = (int)row_team_bytes(p, e->TS, e->layout);
    a.resync = 0;
    x = row_args(p);
    x.penalty_weight = c.penalty_weight;
    x.obj_weight = c.obj_weight > 0 ? c.obj_weight : 1.0;
    x.maximize = c.maximize;
    x.w2 = c.obj_weight2;
    x.mo = e->mo;
  } else {
    a.team_smem = (int)team_bytes_for(kLayouts[e->layout].elem, e->n, e->TS);
    a.resync = kLayouts[e->layout].elem == E_F64;
  }
}

int go_engine_run(go_engine* e, int64_t max_generations, double time_limit_s,
                  go_run_stats* stats) {
  if (!e) return fail(GO_E_INVALID, "null engine");
  if (e->nseq == 0) return fail(GO_E_INVALID, "registry not set");
  CK(cudaSetDevice(e->prob->device));
  const go_engine_config& c = e->cfg;
  go::GlobalState gs{};
  CK(cudaStreamSynchronize(e->stream));  // set_population's copies are asynchronous
  CK(cudaMemcpy(&gs, e->gs, sizeof(gs), cudaMemcpyDeviceToHost));
  long long done = gs.gens_done;
  const unsigned long long rp0 = gs.rd_pos, re0 = gs.rd_elem;
  if (gs.stop) {  // a previous run stopped; resume from the same state
    gs.stop = 0;
    *e->h_stop = 0;
  }
  // history buffer sized for the generations this call may run
  if (e->history_on && max_generations > e->hist_cap) {
    if (e->history) cudaFree(e->history);
    e->hist_cap = std::max<long long>(max_generations, 1);
    CK(cudaMalloc(&e->history, (size_t)e->hist_cap * 8));
  }
  gs.deadline_ns = 0;
  CK(cudaMemcpyAsync(e->gs, &gs, sizeof(gs), cudaMemcpyHostToDevice, e->stream));
  if (time_limit_s > 0) {
    const long long budget = (long long)(time_limit_s * 1e9);
    go::go_arm_deadline_kernel<<<1, 1, 0, e->stream>>>(e->gs, budget);
    CK(cudaGetLastError());
  }
  CK(cudaEventRecord(e->t_start, e->stream));
  long long launches = time_limit_s > 0 ? 1 : 0;  // the deadline kernel
  long long chunk = 0;
  const int I = c.aos_interval, EI = c.elite_interval, MI = c.migration_interval;
  auto next_mult = [](long long g, long long m) { return (g / m + 1) * m; };
  go::EvolveArgs a;
  go::RowArgs x;
  build_evolve_args(e, a, x);
  go::EpilogueArgs q{};
  q.P = e->P;
  q.W = e->W;
  q.genes = e->genes;
  q.scal = e->scal;
  q.pen = e->pen;
  q.best_genes = e->best_genes;
  q.best_scal = e->best_scal;
  q.best_pen = e->best_pen;
  q.best_gen = e->best_gen;
  q.gbest_genes = e->gbest_genes;
  q.scratch = e->scratch;
  q.usage = e->usage;
  q.impr = e->impr;
  q.k_usage = e->k_usage;
  q.k_impr = e->k_impr;
  q.agg = e->agg;
  q.rec_scal = e->rec_scal;
  q.rec_pen = e->rec_pen;
  q.reg = e->reg;
  q.gs = e->gs;
  q.history = e->history_on ? e->history : nullptr;
  q.hist_cap = e->history_on ? e->hist_cap : 0;
  q.host_stop = e->d_stop_map;
  q.pw = c.penalty_weight;
  q.aos_interval = c.aos_interval;
  q.stagnation = c.stagnation_threshold;
  q.alpha = c.aos_alpha;
  q.floor_ = c.aos_floor;
  q.cap = c.aos_cap;
  q.eps = c.aos_eps;
  q.islands = c.islands;
  q.migration = c.migration;
  q.mig_interval = c.migration_interval;
  q.top_n = c.top_n;
  q.elite_interval = c.elite_interval;
  q.has_target = c.has_target;
  q.target = c.target_objective;
  q.obj_sign_over_w = e->obj_sign_over_w;
  q.seed = c.seed;
  q.max_gens = max_generations;
  q.obj2 = e->obj2;
  q.best_obj2 = e->best_obj2;
  q.rec_obj2 = e->rec_obj2;
  q.mo = e->mo;

  double evolve_ms = 0.0;
  long long evolve_launches = 0;
  auto harvest = [&](int s) {
    if (!e->k_pending[s]) return;
    float kms = 0.f;
    if (cudaEventElapsedTime(&kms, e->k_beg[s], e->k_end[s]) == cudaSuccess) evolve_ms += kms;
    e->k_pending[s] = false;
  };
  while (done < max_generations) {
    if (*(volatile int*)e->h_stop) break;
    long long end = std::min<long long>(max_generations, done + go::MAX_CHUNK);
    end = std::min(end, next_mult(done, I));
    end = std::min(end, next_mult(done, EI));
    if (c.islands >= 2) end = std::min(end, next_mult(done, MI));
    if (e->xover && !e->coop) end = done + 1;  // launch boundary = snapshot barrier
    // Lexicographic runs: the global best's genes are taken from the current
    // rows at the end of a one-generation chunk (go_epilogue.cuh)
    if (e->mo.lex) end = done + 1;
    const int slot = (int)(chunk % go_engine::kDepth);
    if (chunk >= go_engine::kDepth) {
      CK(cudaEventSynchronize(e->ring_ev[slot]));
      harvest(slot);
      if (*(volatile int*)e->h_stop) break;
    }
    double* ht = e->h_temps + (size_t)slot * go::MAX_CHUNK;
    for (long long g = done + 1; g <= end; ++g)
      ht[g - done - 1] = c.t0 * std::pow(c.cooling_alpha, (double)(g - 1));  // engine.py:685
    double* dt = e->temps + (size_t)slot * go::MAX_CHUNK;
    CK(cudaMemcpyAsync(dt, ht, (size_t)(end - done) * 8, cudaMemcpyHostToDevice, e->stream));
    a.temps = dt;
    a.gen0 = done + 1;
    a.ngen = (int)(end - done);
    if (e->xover) {  // snapshot of generation gen0 = the population at launch
      CK(cudaMemcpyAsync(e->snap + (size_t)(a.gen0 % go::SNAP_DEPTH) * e->P * e->W, e->genes,
                         (size_t)e->P * e->W * 2, cudaMemcpyDeviceToDevice, e->stream));
      go::go_fill_i32_kernel<<<(e->P + 255) / 256, 256, 0, e->stream>>>(e->prog, e->P,
                                                                        (int)a.gen0);
      CK(cudaGetLastError());
    }
    void* args[] = {&a, &x};
    CK(cudaEventRecord(e->k_beg[slot], e->stream));
    int rc = launch_static_or_jit(e->k_evolve, e->k_evolve_jit, dim3(e->grid), dim3(e->E * e->TS),
                                  e->smem, e->stream, args, e->xover && a.ngen > 1);
    if (rc) return rc;
    CK(cudaEventRecord(e->k_end[slot], e->stream));
    e->k_pending[slot] = true;
    ++evolve_launches;
    q.gen0 = a.gen0;
    q.ngen = a.ngen;
    go::go_epilogue_kernel<<<1, go::EPI_THREADS, 0, e->stream>>>(q);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e->ring_ev[slot], e->stream));
    launches += e->xover ? 3 : 2;  // (+ the snapshot progress fill) evolve, epilogue
    done = end;
    ++chunk;
  }
  CK(cudaEventRecord(e->t_stop, e->stream));
  CK(cudaStreamSynchronize(e->stream));
  for (int s = 0; s < go_engine::kDepth; ++s) harvest(s);
  CK(cudaMemcpy(&gs, e->gs, sizeof(gs), cudaMemcpyDeviceToHost));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e->t_start, e->t_stop));
  e->launches += launches;
  if (stats) {
    stats->generations = gs.gens_done;
    stats->lane_evals = gs.gens_done * (long long)e->P * e->T;
    stats->kernel_launches = launches;
    stats->device_ms = ms;
    stats->stopped_by = gs.stop == 1 ? 1 : (gs.stop == 2 ? 2 : 0);
    stats->error_flags = gs.err;
    stats->reads_pos = (int64_t)(gs.rd_pos - rp0);
    stats->reads_elem = (int64_t)(gs.rd_elem - re0);
    stats->elem_bytes = e->prob->family == 1 ? (e->prob->row_kind == go::RK_QAP ? (int32_t)elem_size(e->prob->elem) : (e->prob->row_kind == go::RK_KNAP ? 8 : 4))
                                             : (int32_t)elem_size(kLayouts[e->layout].elem);
    stats->gene_bytes = 2;
    stats->evolve_ms = evolve_ms;
    stats->evolve_launches = evolve_launches;
  }
  return GO_OK;
}

// One generation of the evolve kernel for every evolver at an explicit
// generation index and temperature, without the epilogue (no global best,
// AOS update, migration or elite injection): the reference's
// evolve_generation (engine.py:538-595) for each evolver.  Each evolver's AOS
// credit of that generation comes back in usage/impr ([P][nseq]) and
// k_usage/k_impr ([P][3]); any pointer may be null.
int go_engine_step(go_engine* e, int64_t generation, double temperature, int32_t* usage,
                   int32_t* impr, int32_t* k_usage, int32_t* k_impr) {
  if (!e) return fail(GO_E_INVALID, "null engine");
  if (e->nseq == 0) return fail(GO_E_INVALID, "registry not set");
  if (generation < 1) return fail(GO_E_INVALID, "generation must be >= 1");
  CK(cudaSetDevice(e->prob->device));
  CK(cudaStreamSynchronize(e->stream));
  go::GlobalState gs{};
  CK(cudaMemcpy(&gs, e->gs, sizeof(gs), cudaMemcpyDeviceToHost));
  gs.stop = 0;
  gs.deadline_ns = 0;
  *e->h_stop = 0;
  CK(cudaMemcpy(e->gs, &gs, sizeof(gs), cudaMemcpyHostToDevice));
  go::EvolveArgs a;
  go::RowArgs x;
  build_evolve_args(e, a, x);
  e->h_temps[0] = temperature;
  CK(cudaMemcpyAsync(e->temps, e->h_temps, 8, cudaMemcpyHostToDevice, e->stream));
  a.temps = e->temps;
  a.gen0 = generation;
  a.ngen = 1;
  if (e->xover) {  // the island snapshot of this generation = the population now
    CK(cudaMemcpyAsync(e->snap + (size_t)(a.gen0 % go::SNAP_DEPTH) * e->P * e->W, e->genes,
                       (size_t)e->P * e->W * 2, cudaMemcpyDeviceToDevice, e->stream));
    go::go_fill_i32_kernel<<<(e->P + 255) / 256, 256, 0, e->stream>>>(e->prog, e->P,
                                                                      (int)a.gen0);
    CK(cudaGetLastError());
  }
  void* args[] = {&a, &x};
  int rc = launch_static_or_jit(e->k_evolve, e->k_evolve_jit, dim3(e->grid), dim3(e->E * e->TS),
                                e->smem, e->stream, args, false);
  if (rc) return rc;
  CK(cudaStreamSynchronize(e->stream));
  e->launches += 1;
  const size_t P = e->P;
  if (usage || impr) {
    std::vector<int> u(P * go::MAX_SEQ), v(P * go::MAX_SEQ);
    CK(cudaMemcpy(u.data(), e->usage, u.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(v.data(), e->impr, v.size() * 4, cudaMemcpyDeviceToHost));
    for (size_t ev = 0; ev < P; ++ev)
      for (int i = 0; i < e->nseq; ++i) {
        if (usage) usage[ev * e->nseq + i] = u[ev * go::MAX_SEQ + i];
        if (impr) impr[ev * e->nseq + i] = v[ev * go::MAX_SEQ + i];
      }
  }
  if (k_usage) CK(cudaMemcpy(k_usage, e->k_usage, P * 3 * 4, cudaMemcpyDeviceToHost));
  if (k_impr) CK(cudaMemcpy(k_impr, e->k_impr, P * 3 * 4, cudaMemcpyDeviceToHost));
  return GO_OK;
}

int go_engine_get_population(go_engine* e, int32_t* genes, int32_t* sizes, double* obj,
                             double* pen) {
  if (!e) return fail(GO_E_INVALID, "null engine");
  CK(cudaSetDevice(e->prob->device));
  const size_t P = e->P, W = e->W;
  const size_t o_g = 0, o_sc = align16(P * W * 2), o_pe = o_sc + P * 8, o_o2 = o_pe + P * 8,
               total = o_o2 + P * 16;
  unsigned char* h = engine_pinned(e, total);
  if (!h) return fail(GO_E_CUDA, "pinned staging allocation failed");
  short* g = (short*)(h + o_g);
  double *sc = (double*)(h + o_sc), *pe = (double*)(h + o_pe), *o2 = (double*)(h + o_o2);
  const cudaStream_t s = e->stream;
  const cudaMemcpyKind D2H = cudaMemcpyDeviceToHost;
  const bool rows = genes || sizes, want_o2 = obj && e->obj2;
  if (rows) CK(cudaMemcpyAsync(g, e->genes, P * W * 2, D2H, s));
  if (obj && !want_o2) CK(cudaMemcpyAsync(sc, e->scal, P * 8, D2H, s));
  if (want_o2) CK(cudaMemcpyAsync(o2, e->obj2, P * 16, D2H, s));
  if (pen) CK(cudaMemcpyAsync(pe, e->pen, P * 8, D2H, s));
  CK(cudaEventRecord(e->pin_ev, s));
  CK(cudaEventSynchronize(e->pin_ev));
  if (rows) from_device_rows(e->prob, g, (int)P, genes, sizes);
  if (want_o2) {
    for (size_t i = 0; i < P; ++i)
      for (int k = 0; k < e->mo.m; ++k) obj[i * e->mo.m + k] = o2[2 * i + k];
  } else if (obj) {
    for (size_t i = 0; i < P; ++i) obj[i] = sc[i] * e->obj_sign_over_w;
  }
  if (pen) std::memcpy(pen, pe, P * 8);
  return GO_OK;
}

int go_engine_get_best(go_engine* e, int32_t* genes, int32_t* sizes, double* obj, double* pen,
                       int64_t* found_gen) {
  if (!e) return fail(GO_E_INVALID, "null engine");
  CK(cudaSetDevice(e->prob->device));
  CK(cudaStreamSynchronize(e->stream));
  go::GlobalState gs{};
  CK(cudaMemcpy(&gs, e->gs, sizeof(gs), cudaMemcpyDeviceToHost));
  std::vector<short> g(e->W);
  const short* src = gs.gev >= 0 ? e->best_genes + (size_t)gs.gev * e->W : e->gbest_genes;
  CK(cudaMemcpy(g.data(), src, (size_t)e->W * 2, cudaMemcpyDeviceToHost));
  from_device_rows(e->prob, g.data(), 1, genes, sizes);
  if (obj && e->obj2) {
    for (int k = 0; k < e->mo.m; ++k) obj[k] = gs.gobj[k];
  } else if (obj) {
    *obj = gs.gscal * e->obj_sign_over_w;
  }
  if (pen) *pen = gs.gpen;
  if (found_gen) *found_gen = gs.ggen;
  return GO_OK;
}

int go_engine_get_registry(go_engine* e, double* weights, double* k_weights, int32_t* stall) {
  if (!e) return fail(GO_E_INVALID, "null engine");
  CK(cudaSetDevice(e->prob->device));
  CK(cudaStreamSynchronize(e->stream));
  go::RegistryDev r;
  CK(cudaMemcpy(&r, e->reg, sizeof(r), cudaMemcpyDeviceToHost));
  if (weights)
    for (int i = 0; i < r.nseq; ++i) weights[i] = r.w[i];
  if (k_weights)
    for (int j = 0; j < 3; ++j) k_weights[j] = r.kw[j];
  if (stall) {
    go::GlobalState gs{};
    CK(cudaMemcpy(&gs, e->gs, sizeof(gs), cudaMemcpyDeviceToHost));
    *stall = (int32_t)gs.stall;
  }
  return GO_OK;
}

int go_engine_get_history(go_engine* e, double* best_phi, int64_t cap, int64_t* count) {
  if (!e) return fail(GO_E_INVALID, "null engine");
  CK(cudaSetDevice(e->prob->device));
  CK(cudaStreamSynchronize(e->stream));
  go::GlobalState gs{};
  CK(cudaMemcpy(&gs, e->gs, sizeof(gs), cudaMemcpyDeviceToHost));
  const long long nh = e->history ? std::min<long long>(gs.hist_count, cap) : 0;
  if (nh > 0) CK(cudaMemcpy(best_phi, e->history, (size_t)nh * 8, cudaMemcpyDeviceToHost));
  if (count) *count = nh;
  return GO_OK;
}

int go_elite_record_bytes(go_engine* e, int64_t* bytes) {
  if (!e || !bytes) return fail(GO_E_INVALID, "bad arguments");
  *bytes = ((int64_t)e->W * 2 + 15) / 16 * 16 + 32;  // {scal, pen, o0, o1} + genes
  return GO_OK;
}

static go::IslandArgs island_args(go_engine* e, void* buf, int top_n) {
  go::IslandArgs a{};
  a.P = e->P;
  a.W = e->W;
  a.genes = e->genes;
  a.scal = e->scal;
  a.pen = e->pen;
  a.gbest_genes = e->gbest_genes;
  a.gs = e->gs;
  a.obj2 = e->obj2;
  a.mo = e->mo;
  a.buf = (unsigned char*)buf;
  int64_t rb = 0;
  go_elite_record_bytes(e, &rb);
  a.rec_bytes = (int)rb;
  a.top_n = top_n;
  a.seed = e->cfg.seed;
  return a;
}

int go_engine_export_elites(go_engine* e, void* device_buf, int top_n) {
  if (!e || !device_buf || top_n < 1 || top_n > 64) return fail(GO_E_INVALID, "bad arguments");
  CK(cudaSetDevice(e->prob->device));
  go::IslandArgs a = island_args(e, device_buf, top_n);
  go::go_export_elites_kernel<<<1, go::EPI_THREADS, 0, e->stream>>>(a);
  CK(cudaGetLastError());
  return GO_OK;
}

int go_engine_import_elites(go_engine* e, const void* device_buf, int n_ranks, int rank,
                            int top_n, int strategy, int64_t event_index) {
  if (!e || !device_buf || n_ranks < 1 || rank < 0 || rank >= n_ranks || top_n < 1 || top_n > 64)
    return fail(GO_E_INVALID, "bad arguments");
  if (strategy == GO_MIG_HYBRID) strategy = event_index % 2 == 0 ? GO_MIG_RING : GO_MIG_GLOBAL_TOP_N;
  CK(cudaSetDevice(e->prob->device));
  go::IslandArgs a = island_args(e, (void*)device_buf, top_n);
  a.n_ranks = n_ranks;
  a.rank = rank;
  a.strategy = strategy;
  a.event = event_index;
  go::go_import_elites_kernel<<<1, go::EPI_THREADS, 0, e->stream>>>(a);
  CK(cudaGetLastError());
  return GO_OK;
}

int go_engine_debug_counters(go_engine* e, int64_t* out, int n) {
  if (!e || !out || n < 1) return fail(GO_E_INVALID, "bad arguments");
  CK(cudaSetDevice(e->prob->device));
  CK(cudaStreamSynchronize(e->stream));
  go::GlobalState gs{};
  CK(cudaMemcpy(&gs, e->gs, sizeof(gs), cudaMemcpyDeviceToHost));
  for (int i = 0; i < n && i < 32; ++i) out[i] = (int64_t)gs.prof[i];
  return GO_OK;
}

int go_engine_stream(go_engine* e, void** stream) {
  if (!e || !stream) return fail(GO_E_INVALID, "bad arguments");
  *stream = (void*)e->stream;
  return GO_OK;
}

int go_engine_sync(go_engine* e) {
  if (!e) return fail(GO_E_INVALID, "null engine");
  CK(cudaStreamSynchronize(e->stream));
  return GO_OK;
}

}  // extern "C"
