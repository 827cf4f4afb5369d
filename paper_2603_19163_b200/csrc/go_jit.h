// go_jit.h — NVRTC compile pipeline for user operators (paper §5.1).
#pragma once
#include <cuda.h>

#include <string>
#include <vector>

namespace gohost {

struct UserOpSrc {
  int id;
  std::string name;
  std::string body;
};

struct JitModule {
  CUmodule mod = nullptr;
  CUfunction evolve = nullptr;
  CUfunction probe = nullptr;
  CUfunction probe_op = nullptr;  // user problems: go_probe_user_op
  std::string key;
  double compile_seconds = 0.0;
  bool cache_hit = false;
};

std::string sha256_hex(const std::string& data);
int jit_max_threads();  // CTA thread cap of JIT-built evolve kernels (GO_EVOLVE_MAX_THREADS)
std::string kernel_dir();

// Builds (or loads from the cubin cache) the evolve + probe kernels of the
// TSP path specialised for distance type `dist_type` with the given user
// operators compiled in as slots 0..n-1.  Returns 0 or a GO_E_* status and a
// compiler log.
// `max_threads` is the kernel's launch bound (GO_EVOLVE_MAX_THREADS; 0 = the
// default jit_max_threads()): teams x lanes per CTA may not exceed it.
int jit_compile_tsp(const std::string& dist_type, const std::vector<UserOpSrc>& ops,
                    std::string* cubin_out, std::string* key_out, bool* hit_out,
                    std::string* log, int max_threads = 0);
int jit_build_tsp(const std::string& dist_type, const std::vector<UserOpSrc>& ops,
                  JitModule* out, std::string* log, int max_threads = 0);

// A user problem: objective / penalty snippet bodies and the named float64
// data arrays they read (byte offsets into the instance image).
struct UserProblemSrc {
  std::string obj, pen, obj2;  // obj2 empty: one objective
  std::vector<std::string> names;
  std::vector<unsigned long long> offsets;
  std::vector<long long> lens;
  std::vector<UserOpSrc> ops;  // user operators, compiled in as slots 0..n-1
  bool rows_global = false;    // lane rows in global memory (long rows)
};
// Builds go_evolve_user (JitModule::evolve) and go_eval_user (JitModule::probe).
int jit_build_user(const UserProblemSrc& up, JitModule* out, std::string* log);

// A built-in row problem's evolve kernel with user operators compiled in:
// kind / element / gene type names as in engine.cu's GO_ROW_KERNEL list.
struct RowOpsSrc {
  std::string kind, elem_type, gene_type;
  bool rows_global = false;
};
int jit_build_rowops(const RowOpsSrc& ro, const std::vector<UserOpSrc>& ops, JitModule* out,
                     std::string* log);

}  // namespace gohost
