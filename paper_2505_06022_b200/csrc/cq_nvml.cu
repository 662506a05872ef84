// SYnergy measurement hooks over NVML (loaded with dlopen so the library
// builds and loads on machines without a driver).
//
// The reference models energy (energy.py:35-71, 150-197); on B200 the
// per-kernel energy is the delta of nvmlDeviceGetTotalEnergyConsumption (mJ)
// around a kernel loop, and the frequency candidates are the supported SM
// clocks.  Locking clocks changes shared hardware state and is refused unless
// CQ_ALLOW_CLOCK_LOCK=1.
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>

#include "cq_common.cuh"

namespace {

typedef int nvmlReturn_t;
typedef struct nvmlDevice_st* nvmlDevice_t;
enum { NVML_SUCCESS = 0, NVML_ERROR_NO_PERMISSION = 4, NVML_ERROR_NOT_SUPPORTED = 3 };
enum { NVML_CLOCK_SM = 1, NVML_CLOCK_MEM = 2 };

struct Nvml {
  void* h = nullptr;
  nvmlReturn_t (*init)(void) = nullptr;
  const char* (*err)(nvmlReturn_t) = nullptr;
  nvmlReturn_t (*by_pci)(const char*, nvmlDevice_t*) = nullptr;
  nvmlReturn_t (*energy)(nvmlDevice_t, unsigned long long*) = nullptr;
  nvmlReturn_t (*power)(nvmlDevice_t, unsigned int*) = nullptr;
  nvmlReturn_t (*clock)(nvmlDevice_t, int, unsigned int*) = nullptr;
  nvmlReturn_t (*max_clock)(nvmlDevice_t, int, unsigned int*) = nullptr;
  nvmlReturn_t (*reasons)(nvmlDevice_t, unsigned long long*) = nullptr;
  nvmlReturn_t (*mem_clocks)(nvmlDevice_t, unsigned int*, unsigned int*) = nullptr;
  nvmlReturn_t (*gfx_clocks)(nvmlDevice_t, unsigned int, unsigned int*, unsigned int*) = nullptr;
  nvmlReturn_t (*lock)(nvmlDevice_t, unsigned int, unsigned int) = nullptr;
  nvmlReturn_t (*unlock)(nvmlDevice_t) = nullptr;
  bool ok = false;
};
Nvml g_nvml;

template <typename F>
void sym(F& f, const char* name) {
  f = reinterpret_cast<F>(dlsym(g_nvml.h, name));
}

int nvml_fail(const char* what, nvmlReturn_t r) {
  cq::set_error("%s: %s", what, g_nvml.err ? g_nvml.err(r) : "nvml error");
  return r == NVML_ERROR_NO_PERMISSION ? CQ_ERR_PERMISSION : CQ_ERR_NVML;
}

int handle(int device, nvmlDevice_t* out) {
  if (!g_nvml.ok) {
    int s = cq_nvml_init();
    if (s != CQ_OK) return s;
  }
  char bus[64];
  CQ_CHECK_CUDA(cudaDeviceGetPCIBusId(bus, sizeof(bus), device));
  nvmlReturn_t r = g_nvml.by_pci(bus, out);
  if (r != NVML_SUCCESS) return nvml_fail("nvmlDeviceGetHandleByPciBusId", r);
  return CQ_OK;
}

}  // namespace

extern "C" {

int cq_nvml_init(void) {
  if (g_nvml.ok) return CQ_OK;
  g_nvml.h = dlopen("libnvidia-ml.so.1", RTLD_NOW | RTLD_GLOBAL);
  if (!g_nvml.h) {
    cq::set_error("dlopen(libnvidia-ml.so.1) failed: %s", dlerror());
    return CQ_ERR_NVML;
  }
  sym(g_nvml.init, "nvmlInit_v2");
  sym(g_nvml.err, "nvmlErrorString");
  sym(g_nvml.by_pci, "nvmlDeviceGetHandleByPciBusId_v2");
  sym(g_nvml.energy, "nvmlDeviceGetTotalEnergyConsumption");
  sym(g_nvml.power, "nvmlDeviceGetPowerUsage");
  sym(g_nvml.clock, "nvmlDeviceGetClockInfo");
  sym(g_nvml.max_clock, "nvmlDeviceGetMaxClockInfo");
  sym(g_nvml.reasons, "nvmlDeviceGetCurrentClocksEventReasons");
  if (!g_nvml.reasons) sym(g_nvml.reasons, "nvmlDeviceGetCurrentClocksThrottleReasons");
  sym(g_nvml.mem_clocks, "nvmlDeviceGetSupportedMemoryClocks");
  sym(g_nvml.gfx_clocks, "nvmlDeviceGetSupportedGraphicsClocks");
  sym(g_nvml.lock, "nvmlDeviceSetGpuLockedClocks");
  sym(g_nvml.unlock, "nvmlDeviceResetGpuLockedClocks");
  if (!g_nvml.init || !g_nvml.by_pci || !g_nvml.energy) {
    cq::set_error("libnvidia-ml.so.1 lacks required symbols");
    return CQ_ERR_NVML;
  }
  nvmlReturn_t r = g_nvml.init();
  if (r != NVML_SUCCESS) return nvml_fail("nvmlInit_v2", r);
  g_nvml.ok = true;
  return CQ_OK;
}

int cq_nvml_energy_mj(int device, uint64_t* mj) {
  nvmlDevice_t h;
  CQ_TRY(handle(device, &h));
  unsigned long long v = 0;
  nvmlReturn_t r = g_nvml.energy(h, &v);
  if (r != NVML_SUCCESS) return nvml_fail("nvmlDeviceGetTotalEnergyConsumption", r);
  *mj = v;
  return CQ_OK;
}

int cq_nvml_power_mw(int device, unsigned int* mw) {
  nvmlDevice_t h;
  CQ_TRY(handle(device, &h));
  nvmlReturn_t r = g_nvml.power(h, mw);
  if (r != NVML_SUCCESS) return nvml_fail("nvmlDeviceGetPowerUsage", r);
  return CQ_OK;
}

int cq_nvml_sm_clock_mhz(int device, unsigned int* current, unsigned int* max) {
  nvmlDevice_t h;
  CQ_TRY(handle(device, &h));
  nvmlReturn_t r = g_nvml.clock(h, NVML_CLOCK_SM, current);
  if (r != NVML_SUCCESS) return nvml_fail("nvmlDeviceGetClockInfo", r);
  r = g_nvml.max_clock(h, NVML_CLOCK_SM, max);
  if (r != NVML_SUCCESS) return nvml_fail("nvmlDeviceGetMaxClockInfo", r);
  return CQ_OK;
}

int cq_nvml_throttle_reasons(int device, unsigned long long* reasons) {
  nvmlDevice_t h;
  CQ_TRY(handle(device, &h));
  if (!g_nvml.reasons) {
    cq::set_error("clock event reasons not available");
    return CQ_ERR_UNSUPPORTED;
  }
  nvmlReturn_t r = g_nvml.reasons(h, reasons);
  if (r != NVML_SUCCESS) return nvml_fail("nvmlDeviceGetCurrentClocksEventReasons", r);
  return CQ_OK;
}

int cq_nvml_supported_sm_clocks(int device, unsigned int* mhz, int* count) {
  nvmlDevice_t h;
  CQ_TRY(handle(device, &h));
  unsigned int nmem = 16, mems[16];
  nvmlReturn_t r = g_nvml.mem_clocks(h, &nmem, mems);
  if (r != NVML_SUCCESS) return nvml_fail("nvmlDeviceGetSupportedMemoryClocks", r);
  unsigned int n = (unsigned int)*count;
  r = g_nvml.gfx_clocks(h, mems[0], &n, mhz);
  if (r != NVML_SUCCESS) return nvml_fail("nvmlDeviceGetSupportedGraphicsClocks", r);
  *count = (int)n;
  return CQ_OK;
}

static bool clock_lock_allowed() {
  const char* v = getenv("CQ_ALLOW_CLOCK_LOCK");
  return v && strcmp(v, "1") == 0;
}

int cq_nvml_lock_sm_clock(int device, unsigned int mhz) {
  if (!clock_lock_allowed()) {
    cq::set_error("SM clock locking is disabled (set CQ_ALLOW_CLOCK_LOCK=1 on a machine you own)");
    return CQ_ERR_PERMISSION;
  }
  nvmlDevice_t h;
  CQ_TRY(handle(device, &h));
  nvmlReturn_t r = g_nvml.lock(h, mhz, mhz);
  if (r != NVML_SUCCESS) return nvml_fail("nvmlDeviceSetGpuLockedClocks", r);
  return CQ_OK;
}

int cq_nvml_reset_sm_clock(int device) {
  if (!clock_lock_allowed()) {
    cq::set_error("SM clock locking is disabled (set CQ_ALLOW_CLOCK_LOCK=1 on a machine you own)");
    return CQ_ERR_PERMISSION;
  }
  nvmlDevice_t h;
  CQ_TRY(handle(device, &h));
  nvmlReturn_t r = g_nvml.unlock(h);
  if (r != NVML_SUCCESS) return nvml_fail("nvmlDeviceResetGpuLockedClocks", r);
  return CQ_OK;
}

}  // extern "C"
