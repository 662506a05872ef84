// Shared helpers of libcq: error reporting, per-device state.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/cq.h"

namespace cq {

void set_error(const char* fmt, ...);

struct DeviceState {
  bool ready = false;
  cudaStream_t streams[CQ_NUM_STREAMS] = {};
  int* error_flag = nullptr;        // [0]=code, [1..6]=point (int64 as 2x int32), device memory
  int sm_count = 0;
  int64_t l2_bytes = 0;
};

DeviceState* device_state(int device);  // nullptr if not initialised
int ensure_device(int device);           // initialise on first use
cudaStream_t stream_of(int device, int stream);
// Grow-only scratch per (device, stream, slot): reused across launches so a
// captured CUDA graph holds no allocation nodes.  Stream-ordered use only.
int scratch(int device, int stream, int slot, size_t bytes, void** ptr);

}  // namespace cq

#define CQ_CHECK_CUDA(expr)                                                          \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      cq::set_error("%s:%d: %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return CQ_ERR_CUDA;                                                            \
    }                                                                                \
  } while (0)

#define CQ_CHECK_LAUNCH()                                                            \
  do {                                                                               \
    cudaError_t _e = cudaGetLastError();                                             \
    if (_e != cudaSuccess) {                                                         \
      cq::set_error("%s:%d: kernel launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return CQ_ERR_CUDA;                                                            \
    }                                                                                \
  } while (0)

#define CQ_REQUIRE(cond, ...)                                                        \
  do {                                                                               \
    if (!(cond)) {                                                                   \
      cq::set_error(__VA_ARGS__);                                                    \
      return CQ_ERR_ARG;                                                             \
    }                                                                                \
  } while (0)

#define CQ_TRY(expr)                \
  do {                              \
    int _s = (expr);                \
    if (_s != CQ_OK) return _s;     \
  } while (0)
