// go_jit.cpp — NVRTC pipeline: user operator snippets -> sm_100a cubin.
//
// Mirrors the paper's JIT pipeline (§5.1): the operator code is
// injected into the framework's kernel template (here: a `UserOps` switch
// that go_evolve_perm.cuh dispatches sequence ids >= 100 to), compiled for
// sm_100a, and cached on disk under the SHA-256 of the full source, the
// framework headers and the options (first build seconds, cache hit ~ms).
#include "go_jit.h"

#include "go_drv.h"

#include <dlfcn.h>
#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>

#include "../../include/cugenopt.h"

namespace gohost {

// ---- SHA-256 (FIPS 180-4) ---------------------------------------------------
namespace {
const uint32_t K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4,
    0xab1c5ed5, 0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe,
    0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f,
    0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7,
    0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc,
    0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b,
    0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116,
    0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
    0xc67178f2};

inline uint32_t rotr(uint32_t x, int r) { return (x >> r) | (x << (32 - r)); }

void sha_block(uint32_t h[8], const unsigned char* p) {
  uint32_t w[64];
  for (int i = 0; i < 16; ++i)
    w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 | (uint32_t)p[4 * i + 2] << 8 |
           p[4 * i + 3];
  for (int i = 16; i < 64; ++i) {
    const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
    const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
    w[i] = w[i - 16] + s0 + w[i - 7] + s1;
  }
  uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
  for (int i = 0; i < 64; ++i) {
    const uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
    const uint32_t ch = (e & f) ^ (~e & g);
    const uint32_t t1 = hh + S1 + ch + K256[i] + w[i];
    const uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
    const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
    const uint32_t t2 = S0 + mj;
    hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
  }
  h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}
}  // namespace

std::string sha256_hex(const std::string& data) {
  uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                   0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  std::string m = data;
  const uint64_t bits = (uint64_t)data.size() * 8;
  m.push_back((char)0x80);
  while (m.size() % 64 != 56) m.push_back(0);
  for (int i = 7; i >= 0; --i) m.push_back((char)(bits >> (8 * i)));
  for (size_t off = 0; off < m.size(); off += 64) sha_block(h, (const unsigned char*)m.data() + off);
  char out[65];
  for (int i = 0; i < 8; ++i) snprintf(out + 8 * i, 9, "%08x", h[i]);
  return std::string(out, 64);
}

static std::string read_file(const std::string& path, bool* ok) {
  std::ifstream f(path, std::ios::binary);
  if (!f) {
    *ok = false;
    return "";
  }
  std::stringstream ss;
  ss << f.rdbuf();
  *ok = true;
  return ss.str();
}

std::string kernel_dir() {
  if (const char* env = getenv("GO_KERNEL_DIR")) return env;
  Dl_info info;
  if (dladdr((void*)&kernel_dir, &info) && info.dli_fname) {
    std::string so = info.dli_fname;
    const size_t slash = so.rfind('/');
    const std::string dir = slash == std::string::npos ? "." : so.substr(0, slash);
    return dir + "/../csrc/kernels";
  }
  return "paper_2603_19163_b200/csrc/kernels";
}

static std::string cache_dir() {
  std::string d;
  if (const char* env = getenv("GO_JIT_CACHE")) d = env;
  else if (const char* home = getenv("HOME")) d = std::string(home) + "/.cache/cugenopt";
  else d = "/tmp/cugenopt-cache";
  std::string acc;
  std::stringstream ss(d);
  std::string part;
  if (!d.empty() && d[0] == '/') acc = "";
  while (std::getline(ss, part, '/')) {
    if (part.empty()) continue;
    acc += "/" + part;
    mkdir(acc.c_str(), 0755);
  }
  return d;
}

// 384 threads = 3 teams of 128 lanes per CTA, 168 registers per thread: the
// C2 shared-memory budget (int16 triangle + per-warp scratch rows) holds 3
// teams, and the register headroom removes most of the 128-register spills
// (C2: 84.8 M vs 76.8 M move evals/s at 512, profiles/r02_*).
int jit_max_threads() {
  const char* e = getenv("GO_EVOLVE_MAX_THREADS");
  const int v = e ? atoi(e) : 384;
  return (v >= 128 && v <= 1024 && v % 32 == 0) ? v : 384;
}

static const char* kHeaders[] = {"go_common.cuh",      "go_dist.cuh",      "go_perm.cuh",
                                 "go_perm_lns.cuh",    "go_args.cuh",      "go_evolve_perm.cuh",
                                 "go_tsp_entry.cuh",   "go_row.cuh",       "go_part.cuh",
                                 "go_evolve_row.cuh",  "go_row_entry.cuh"};

// NVRTC compile of a generated translation unit (plus the user snippets it
// #line-references) with the SHA-256 cubin cache.
static int jit_compile_source(const std::string& source, const std::vector<UserOpSrc>& ops,
                              std::string* cubin_out, std::string* key_out, bool* hit_out,
                              std::string* log, int max_threads = 0) {

  const std::string kdir = kernel_dir();
  std::string headers_blob;
  for (const char* h : kHeaders) {
    bool ok = false;
    headers_blob += read_file(kdir + "/" + h, &ok);
    if (!ok) {
      *log = "cannot read framework header " + kdir + "/" + h;
      return GO_E_COMPILE;
    }
  }
  const std::string inc = "-I" + kdir;
  const char* extra = getenv("GO_JIT_DEFINE");  // e.g. GO_PHASE_TIMING (profiling builds)
  const std::string extra_opt = std::string("-D") + (extra && *extra ? extra : "GO_JIT_DEFAULT=1");
  const std::string thr_opt = "-DGO_EVOLVE_MAX_THREADS=" +
                              std::to_string(max_threads > 0 ? max_threads : jit_max_threads());
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false", "-lineinfo",
                        "-default-device", "-DGO_JIT=1", extra_opt.c_str(), thr_opt.c_str(),
                        inc.c_str()};
  const int nopts = sizeof(opts) / sizeof(opts[0]);
  std::string keyblob = source + headers_blob;
  for (int i = 0; i < nopts - 1; ++i) keyblob += opts[i];
  int ver_major = 0, ver_minor = 0;
  nvrtcVersion(&ver_major, &ver_minor);
  keyblob += std::to_string(ver_major) + "." + std::to_string(ver_minor);
  *key_out = sha256_hex(keyblob);
  const std::string cdir = cache_dir();
  const std::string path = cdir + "/" + *key_out + ".cubin";
  // The generated translation unit and each operator snippet are written next
  // to the cubin and referenced by #line, so compiler errors name the operator
  // and ncu's source page can import them.
  const std::string opdir = cdir + "/" + *key_out + ".ops";
  mkdir(opdir.c_str(), 0755);
  std::string final_src = source;
  for (size_t at = final_src.find("@OPDIR@"); at != std::string::npos;
       at = final_src.find("@OPDIR@", at))
    final_src.replace(at, 7, opdir);
  for (const auto& op : ops) {
    std::ofstream f(opdir + "/" + op.name + ".cuh");
    f << op.body;
  }
  const std::string src_path = opdir + "/go_user_ops.cu";
  {
    std::ofstream f(src_path);
    f << final_src;
  }

  bool hit = false;
  std::string cubin = read_file(path, &hit);
  if (!hit || cubin.empty()) {
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, final_src.c_str(), src_path.c_str(), 0, nullptr, nullptr) !=
        NVRTC_SUCCESS) {
      *log = "nvrtcCreateProgram failed";
      return GO_E_COMPILE;
    }
    const nvrtcResult rc = nvrtcCompileProgram(prog, nopts, opts);
    size_t lsz = 0;
    nvrtcGetProgramLogSize(prog, &lsz);
    std::string plog(lsz, '\0');
    if (lsz) nvrtcGetProgramLog(prog, &plog[0]);
    if (rc != NVRTC_SUCCESS) {
      *log = plog;
      nvrtcDestroyProgram(&prog);
      return GO_E_COMPILE;
    }
    size_t csz = 0;
    nvrtcGetCUBINSize(prog, &csz);
    cubin.resize(csz);
    nvrtcGetCUBIN(prog, &cubin[0]);
    nvrtcDestroyProgram(&prog);
    const std::string tmp = path + ".tmp." + std::to_string(getpid());
    std::ofstream f(tmp, std::ios::binary);
    f.write(cubin.data(), (std::streamsize)cubin.size());
    f.close();
    rename(tmp.c_str(), path.c_str());
  }
  *hit_out = hit;
  *cubin_out = cubin;
  return GO_OK;
}

int jit_compile_tsp(const std::string& dist_type, const std::vector<UserOpSrc>& ops,
                    std::string* cubin_out, std::string* key_out, bool* hit_out,
                    std::string* log, int max_threads) {
  std::ostringstream src;
  src << "// generated by go_jit.cpp — user operators for the TSP evolve kernel\n"
      << "#include \"go_tsp_entry.cuh\"\n"
      << "namespace go { namespace user {\n";
  for (size_t i = 0; i < ops.size(); ++i) {
    src << "// operator " << ops[i].id << " (" << ops[i].name << ")\n"
        << "template <class Ctx> __device__ __forceinline__ void op_slot" << i
        << "(Ctx& ctx) {\n#line 1 \"@OPDIR@/" << ops[i].name << ".cuh\"\n"
        << ops[i].body << "\n}\n";
  }
  src << "}  // namespace user\nstruct UserOps {\n"
      << "  template <class Ctx> __device__ __forceinline__ static void run(int slot, Ctx& ctx) {\n"
      << "    switch (slot) {\n";
  for (size_t i = 0; i < ops.size(); ++i)
    src << "      case " << i << ": user::op_slot" << i << "(ctx); break;\n";
  src << "      default: ctx.err |= ERR_UNKNOWN_SEQ;\n    }\n  }\n};\n}  // namespace go\n"
      << "GO_TSP_KERNELS(jit, " << dist_type << ", go::UserOps)\n";
  return jit_compile_source(src.str(), ops, cubin_out, key_out, hit_out, log, max_threads);
}

int jit_build_tsp(const std::string& dist_type, const std::vector<UserOpSrc>& ops,
                  JitModule* out, std::string* log, int max_threads) {
  const auto t0 = std::chrono::steady_clock::now();
  std::string cubin;
  bool hit = false;
  const int rc = jit_compile_tsp(dist_type, ops, &cubin, &out->key, &hit, log, max_threads);
  if (rc) return rc;
  const Drv* d = drv();
  if (!d) {
    *log = "CUDA driver API unavailable";
    return GO_E_NODEVICE;
  }
  CUresult cr = d->ModuleLoadData(&out->mod, cubin.data());
  if (cr != CUDA_SUCCESS) {
    const char* s = nullptr;
    d->GetErrorString(cr, &s);
    *log = std::string("cuModuleLoadData: ") + (s ? s : "?");
    return GO_E_CUDA;
  }
  if (d->ModuleGetFunction(&out->evolve, out->mod, "go_evolve_tsp_jit") != CUDA_SUCCESS ||
      d->ModuleGetFunction(&out->probe, out->mod, "go_probe_tsp_jit") != CUDA_SUCCESS) {
    *log = "JIT module lacks go_evolve_tsp_jit / go_probe_tsp_jit";
    return GO_E_COMPILE;
  }
  out->cache_hit = hit;
  out->compile_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return GO_OK;
}

// ---- user problems: NVRTC-compiled objective / penalty ----------
int jit_build_user(const UserProblemSrc& up, JitModule* out, std::string* log) {
  const auto t0 = std::chrono::steady_clock::now();
  std::ostringstream src;
  src << "// generated by go_jit.cpp — user problem (objective + penalty snippets)\n"
      << "#include \"go_row_entry.cuh\"\n"
      << "namespace go { namespace user {\n"
      << "struct Data {\n";
  for (size_t i = 0; i < up.names.size(); ++i)
    src << "  const double* " << up.names[i] << ";\n  int " << up.names[i] << "_len;\n";
  src << "  int _unused;\n};\n"
      << "__device__ __forceinline__ Data make_data(const unsigned char* b) {\n  Data d;\n";
  for (size_t i = 0; i < up.names.size(); ++i)
    src << "  d." << up.names[i] << " = (const double*)(b + " << up.offsets[i] << "ull);\n"
        << "  d." << up.names[i] << "_len = " << up.lens[i] << ";\n";
  src << "  d._unused = 0;\n  return d;\n}\n"
      << "template <class Sol> __device__ __forceinline__ double compute_obj(const Sol& sol, "
         "const Data& data) {\n#line 1 \"@OPDIR@/compute_obj.cuh\"\n"
      << up.obj << "\n}\n"
      << "template <class Sol> __device__ __forceinline__ double compute_penalty(const Sol& sol, "
         "const Data& data) {\n#line 1 \"@OPDIR@/compute_penalty.cuh\"\n"
      << (up.pen.empty() ? std::string("return 0.0;") : up.pen) << "\n}\n"
      << "template <class Sol> __device__ __forceinline__ double compute_obj2(const Sol& sol, "
         "const Data& data) {\n#line 1 \"@OPDIR@/compute_obj2.cuh\"\n"
      << (up.obj2.empty() ? std::string("return 0.0;") : up.obj2) << "\n}\n";
  for (size_t i = 0; i < up.ops.size(); ++i)
    src << "// user operator " << up.ops[i].id << " (" << up.ops[i].name << ")\n"
        << "template <class Ctx> __device__ __forceinline__ void op_slot" << i
        << "(Ctx& ctx, const Data& data) {\n#line 1 \"@OPDIR@/" << up.ops[i].name << ".cuh\"\n"
        << up.ops[i].body << "\n}\n";
  src << "}  // namespace user\n"
      << "struct UserProblem {\n  static constexpr bool kHasOps = true;\n"
      << "  template <class C> __device__ __forceinline__ static void op(int slot, C& ctx, "
         "const unsigned char* b) {\n"
      << "    const user::Data data = user::make_data(b);\n    (void)data;\n    switch (slot) {\n";
  for (size_t i = 0; i < up.ops.size(); ++i)
    src << "      case " << i << ": user::op_slot" << i << "(ctx, data); break;\n";
  src << "      default: ctx.err() |= ERR_UNKNOWN_SEQ;\n    }\n  }\n"
      << "  static constexpr int kObjectives = " << (up.obj2.empty() ? 1 : 2) << ";\n"
      << "  template <class S> __device__ __forceinline__ static double obj2(const S& s, "
         "const unsigned char* b) { return user::compute_obj2(s, user::make_data(b)); }\n"
      << "  template <class S> __device__ __forceinline__ static double obj(const S& s, "
         "const unsigned char* b) { return user::compute_obj(s, user::make_data(b)); }\n"
      << "  template <class S> __device__ __forceinline__ static double pen(const S& s, "
         "const unsigned char* b) { return user::compute_penalty(s, user::make_data(b)); }\n"
      << "};\n}  // namespace go\nGO_USER_KERNELS_RG(go::UserProblem, "
      << (up.rows_global ? "true" : "false") << ")\n";
  std::vector<UserOpSrc> files = {{0, "compute_obj", up.obj},
                                  {1, "compute_penalty", up.pen.empty() ? "return 0.0;" : up.pen}};
  if (!up.obj2.empty()) files.push_back({2, "compute_obj2", up.obj2});
  for (const auto& op : up.ops) files.push_back(op);
  std::string cubin;
  bool hit = false;
  int rc = jit_compile_source(src.str(), files, &cubin, &out->key, &hit, log);
  if (rc) return rc;
  const Drv* d = drv();
  if (!d) {
    *log = "CUDA driver API unavailable";
    return GO_E_NODEVICE;
  }
  CUresult cr = d->ModuleLoadData(&out->mod, cubin.data());
  if (cr != CUDA_SUCCESS) {
    const char* s = nullptr;
    d->GetErrorString(cr, &s);
    *log = std::string("cuModuleLoadData: ") + (s ? s : "?");
    return GO_E_CUDA;
  }
  if (d->ModuleGetFunction(&out->evolve, out->mod, "go_evolve_user") != CUDA_SUCCESS ||
      d->ModuleGetFunction(&out->probe, out->mod, "go_eval_user") != CUDA_SUCCESS ||
      d->ModuleGetFunction(&out->probe_op, out->mod, "go_probe_user_op") != CUDA_SUCCESS) {
    *log = "JIT module lacks go_evolve_user / go_eval_user / go_probe_user_op";
    return GO_E_COMPILE;
  }
  out->cache_hit = hit;
  out->compile_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return GO_OK;
}

// ---- user operators on the built-in row kernels (QAP / knapsack / JSP-int /
// partition problems): the hand-written evolve kernel of `kind` instantiated
// with the operators as U::op slots (register_custom, operators.py:634-669)
int jit_build_rowops(const RowOpsSrc& ro, const std::vector<UserOpSrc>& ops, JitModule* out,
                     std::string* log) {
  const auto t0 = std::chrono::steady_clock::now();
  std::ostringstream src;
  src << "// generated by go_jit.cpp — user operators on a built-in row problem\n"
      << "#include \"go_row_entry.cuh\"\n"
      << "namespace go { namespace user {\n";
  for (size_t i = 0; i < ops.size(); ++i)
    src << "// user operator " << ops[i].id << " (" << ops[i].name << ")\n"
        << "template <class Ctx> __device__ __forceinline__ void op_slot" << i
        << "(Ctx& ctx) {\n#line 1 \"@OPDIR@/" << ops[i].name << ".cuh\"\n" << ops[i].body
        << "\n}\n";
  src << "}  // namespace user\n"
      << "struct RowUserOps : NoUser {\n  static constexpr bool kHasOps = true;\n"
      << "  template <class C> __device__ __forceinline__ static void op(int slot, C& ctx, "
         "const unsigned char*) {\n    switch (slot) {\n";
  for (size_t i = 0; i < ops.size(); ++i)
    src << "      case " << i << ": user::op_slot" << i << "(ctx); break;\n";
  src << "      default: ctx.err() |= ERR_UNKNOWN_SEQ;\n    }\n  }\n};\n}  // namespace go\n"
      << "GO_ROWOPS_KERNELS(" << ro.kind << ", " << ro.elem_type << ", " << ro.gene_type
      << ", go::RowUserOps, " << (ro.rows_global ? "true" : "false") << ")\n";
  std::string cubin;
  bool hit = false;
  int rc = jit_compile_source(src.str(), ops, &cubin, &out->key, &hit, log);
  if (rc) return rc;
  const Drv* d = drv();
  if (!d) {
    *log = "CUDA driver API unavailable";
    return GO_E_NODEVICE;
  }
  CUresult cr = d->ModuleLoadData(&out->mod, cubin.data());
  if (cr != CUDA_SUCCESS) {
    const char* es = nullptr;
    d->GetErrorString(cr, &es);
    *log = std::string("cuModuleLoadData: ") + (es ? es : "?");
    return GO_E_CUDA;
  }
  if (d->ModuleGetFunction(&out->evolve, out->mod, "go_evolve_rowops") != CUDA_SUCCESS ||
      d->ModuleGetFunction(&out->probe_op, out->mod, "go_probe_rowop") != CUDA_SUCCESS) {
    *log = "JIT module lacks go_evolve_rowops / go_probe_rowop";
    return GO_E_COMPILE;
  }
  out->cache_hit = hit;
  out->compile_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return GO_OK;
}

}  // namespace gohost
