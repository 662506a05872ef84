// DSL -> CUDA JIT: NVRTC compiles a task body, lowered by the host
// (paper_2505_06022_b200/jit.py) to straight-line sm_100a code, and the
// kernel takes the same cq_expr_t parameter block as the device interpreter
// (cq_kernels.cu, expr_kernel), so both produce identical bits -- one IEEE
// rounding per DSL operator in tree order (reference kernel.py:291-331).
// any clusterq body at compiled-kernel speed.
#include <cuda.h>
#include <nvrtc.h>

#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "cq_common.cuh"

namespace {

struct Jit {
  std::vector<char> cubin;
  std::string name;
  std::map<int, CUfunction> fn;  // per device
};

std::mutex g_jit_mu;
std::vector<Jit*> g_jits;

typedef CUresult (*PFN_load)(CUmodule*, const void*);
typedef CUresult (*PFN_getfn)(CUfunction*, CUmodule, const char*);
typedef CUresult (*PFN_launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                               CUstream, void**, void**);
typedef CUresult (*PFN_setattr)(CUfunction, CUfunction_attribute, int);

template <typename F>
F driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}

}  // namespace

extern "C" {

int cq_jit_compile(const char* source, const char* kernel_name, int n_headers, const char** header_src,
                   const char** header_names, uint64_t* handle) {
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, source, "cq_jit.cu", n_headers, header_src, header_names) != NVRTC_SUCCESS) {
    cq::set_error("nvrtcCreateProgram failed");
    return CQ_ERR_CUDA;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-default-device", "--fmad=false"};
  nvrtcResult r = nvrtcCompileProgram(prog, 4, opts);
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    nvrtcDestroyProgram(&prog);
    cq::set_error("nvrtc: %s", log.c_str());
    return CQ_ERR_CUDA;
  }
  size_t size = 0;
  nvrtcGetCUBINSize(prog, &size);
  Jit* j = new Jit();
  j->cubin.resize(size);
  nvrtcGetCUBIN(prog, j->cubin.data());
  nvrtcDestroyProgram(&prog);
  j->name = kernel_name;
  std::lock_guard<std::mutex> lk(g_jit_mu);
  g_jits.push_back(j);
  *handle = (uint64_t)g_jits.size();
  return CQ_OK;
}

int cq_jit_launch(uint64_t handle, int device, int stream, const cq_expr_t* expr) {
  CQ_TRY(cq::ensure_device(device));
  cudaStream_t st = cq::stream_of(device, stream);
  CQ_REQUIRE(st != nullptr, "bad stream %d", stream);
  CQ_REQUIRE(handle >= 1 && handle <= g_jits.size(), "unknown jit handle");
  CQ_CHECK_CUDA(cudaSetDevice(device));
  Jit* j = g_jits[handle - 1];
  CUfunction f;
  {
    std::lock_guard<std::mutex> lk(g_jit_mu);
    auto it = j->fn.find(device);
    if (it == j->fn.end()) {
      static PFN_load load = driver_fn<PFN_load>("cuModuleLoadData");
      static PFN_getfn getfn = driver_fn<PFN_getfn>("cuModuleGetFunction");
      CQ_REQUIRE(load && getfn, "driver module API unavailable");
      CUmodule mod;
      if (load(&mod, j->cubin.data()) != CUDA_SUCCESS || getfn(&f, mod, j->name.c_str()) != CUDA_SUCCESS) {
        cq::set_error("cuModuleLoadData/GetFunction failed for %s", j->name.c_str());
        return CQ_ERR_CUDA;
      }
      j->fn[device] = f;
    } else {
      f = it->second;
    }
  }
  static PFN_launch launch = driver_fn<PFN_launch>("cuLaunchKernel");
  CQ_REQUIRE(launch, "cuLaunchKernel unavailable");
  int64_t vol = 1;
  for (int k = 0; k < CQ_MAX_DIMS; ++k) vol *= expr->box.hi[k] - expr->box.lo[k];
  if (vol <= 0) return CQ_OK;
  cq::DeviceState* ds = cq::device_state(device);
  int64_t blocks = (vol + 255) / 256;
  int64_t cap = (int64_t)ds->sm_count * 16;
  unsigned grid = (unsigned)(blocks < cap ? blocks : cap);
  void* flag = ds->error_flag;
  void* params[] = {const_cast<cq_expr_t*>(expr), &flag};
  if (launch(f, grid, 1, 1, 256, 1, 1, 0, (CUstream)st, params, nullptr) != CUDA_SUCCESS) {
    cq::set_error("cuLaunchKernel failed for %s", j->name.c_str());
    return CQ_ERR_CUDA;
  }
  return CQ_OK;
}

}  // extern "C"
