// go_drv.h — driver-API entry points resolved through the CUDA runtime
// (cudaGetDriverEntryPoint), so libcugenopt.so does not link libcuda and
// loads (and exports its ABI) on machines without a driver; device calls
// then fail with GO_E_NODEVICE instead of the loader refusing the library.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace gohost {

struct Drv {
  CUresult (*ModuleLoadData)(CUmodule*, const void*) = nullptr;
  CUresult (*ModuleUnload)(CUmodule) = nullptr;
  CUresult (*ModuleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                           unsigned, CUstream, void**, void**) = nullptr;
  CUresult (*LaunchCooperativeKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned,
                                      unsigned, unsigned, CUstream, void**) = nullptr;
  CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*OccupancyMaxActiveBlocksPerMultiprocessor)(int*, CUfunction, int, size_t) = nullptr;
  CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
  bool ok = false;
};

// Resolves once; returns nullptr when no driver is present.
inline const Drv* drv() {
  static Drv d;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    bool ok = true;
#define GO_RESOLVE(field, sym)                                                              \
  ok = ok && cudaGetDriverEntryPoint(sym, (void**)&d.field, cudaEnableDefault, &q) ==       \
                 cudaSuccess && q == cudaDriverEntryPointSuccess && d.field != nullptr
    GO_RESOLVE(ModuleLoadData, "cuModuleLoadData");
    GO_RESOLVE(ModuleUnload, "cuModuleUnload");
    GO_RESOLVE(ModuleGetFunction, "cuModuleGetFunction");
    GO_RESOLVE(LaunchKernel, "cuLaunchKernel");
    GO_RESOLVE(LaunchCooperativeKernel, "cuLaunchCooperativeKernel");
    GO_RESOLVE(FuncSetAttribute, "cuFuncSetAttribute");
    GO_RESOLVE(OccupancyMaxActiveBlocksPerMultiprocessor,
               "cuOccupancyMaxActiveBlocksPerMultiprocessor");
    GO_RESOLVE(GetErrorString, "cuGetErrorString");
#undef GO_RESOLVE
    d.ok = ok;
  }
  return d.ok ? &d : nullptr;
}

}  // namespace gohost
