// libcq runtime: device state, pooled allocation, copies, events, NCCL.
//
// Replaces the data-movement side of the reference simulator
// (pkg/src/clusterq/simulator.py:81-98 per-node storage, :166-193 push /
// await-push payloads, :210-222 final gather) with HBM allocations, DMA
// copies over PCIe / NVLink and NCCL point-to-point transfers.
#include <cstring>
#include <nccl.h>

#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "cq_common.cuh"

namespace cq {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static const int kMaxDevices = 64;
static DeviceState g_dev[kMaxDevices];
static std::mutex g_mu;

DeviceState* device_state(int device) {
  if (device < 0 || device >= kMaxDevices || !g_dev[device].ready) return nullptr;
  return &g_dev[device];
}

int ensure_device(int device) {
  if (device < 0 || device >= kMaxDevices) {
    set_error("device %d out of range", device);
    return CQ_ERR_ARG;
  }
  DeviceState& d = g_dev[device];
  if (d.ready) return CQ_OK;
  std::lock_guard<std::mutex> lk(g_mu);
  if (d.ready) return CQ_OK;
  CQ_CHECK_CUDA(cudaSetDevice(device));
  int lo = 0, hi = 0;
  CQ_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  // compute: default priority; boundary (halo rows): highest; comm: highest.
  CQ_CHECK_CUDA(cudaStreamCreateWithPriority(&d.streams[CQ_STREAM_COMPUTE], cudaStreamNonBlocking, lo));
  CQ_CHECK_CUDA(cudaStreamCreateWithPriority(&d.streams[CQ_STREAM_BOUNDARY], cudaStreamNonBlocking, hi));
  CQ_CHECK_CUDA(cudaStreamCreateWithPriority(&d.streams[CQ_STREAM_COMM], cudaStreamNonBlocking, hi));
  for (int l = 0; l < CQ_NUM_LANES; ++l)
    CQ_CHECK_CUDA(cudaStreamCreateWithPriority(&d.streams[CQ_STREAM_LANE0 + l], cudaStreamNonBlocking, lo));
  CQ_CHECK_CUDA(cudaMalloc(&d.error_flag, 8 * sizeof(int)));
  // error key all-ones == "no error" (atomicMin records the first failure)
  CQ_CHECK_CUDA(cudaMemset(d.error_flag, 0xff, 2 * sizeof(int)));
  // stream-ordered scratch (cudaMallocAsync in the GEMM split pass) keeps its
  // physical memory between replays instead of re-mapping it every call
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  cudaDeviceProp prop;
  CQ_CHECK_CUDA(cudaGetDeviceProperties(&prop, device));
  d.sm_count = prop.multiProcessorCount;
  d.l2_bytes = prop.l2CacheSize;
  d.ready = true;
  return CQ_OK;
}

cudaStream_t stream_of(int device, int stream) {
  DeviceState* d = device_state(device);
  if (!d || stream < 0 || stream >= CQ_NUM_STREAMS) return nullptr;
  return d->streams[stream];
}

// Per (device, stream, slot) scratch that only grows.  A grown-out block is
// retired, not freed: queued work or an already captured CUDA graph may
// still reference it (freeing it would need a stream synchronize, illegal
// while capturing, and would still break the graph); retired blocks are
// freed by cq_shutdown after a device synchronize.  Growth during a capture
// is refused -- the run before the capture sizes every scratch.
static std::map<std::tuple<int, int, int>, std::pair<void*, size_t>> g_scratch;
static std::vector<std::pair<int, void*>> g_retired;

int scratch(int device, int stream, int slot, size_t bytes, void** ptr) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto& e = g_scratch[std::make_tuple(device, stream, slot)];
  if (e.second < bytes) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CQ_CHECK_CUDA(cudaStreamIsCapturing(stream_of(device, stream), &cap));
    CQ_REQUIRE(cap == cudaStreamCaptureStatusNone,
               "scratch: growing slot %d to %zu bytes while capturing a CUDA graph (run the plan once "
               "before capturing it)", slot, bytes);
    if (e.first) g_retired.emplace_back(device, e.first);
    e.first = nullptr;
    e.second = 0;
    CQ_CHECK_CUDA(cudaMalloc(&e.first, bytes));
    e.second = bytes;
  }
  *ptr = e.first;
  return CQ_OK;
}

static void free_scratch(int device) {
  for (auto it = g_scratch.begin(); it != g_scratch.end();) {
    if (std::get<0>(it->first) == device) {
      cudaFree(it->second.first);
      it = g_scratch.erase(it);
    } else {
      ++it;
    }
  }
  for (auto it = g_retired.begin(); it != g_retired.end();) {
    if (it->first == device) {
      cudaFree(it->second);
      it = g_retired.erase(it);
    } else {
      ++it;
    }
  }
}

// ------------------------------------------------------------- memory pool
// Exact-size free lists per device: repeated runs of the same plan reuse the
// same blocks without cudaMalloc/cudaFree on the critical path.
struct Pool {
  std::multimap<int64_t, void*> free_blocks;
  std::unordered_map<void*, int64_t> live;
};
static Pool g_pool[kMaxDevices];

}  // namespace cq

using namespace cq;

#define CQ_STREAM(dev, s)                                                   \
  cudaStream_t st = stream_of(dev, s);                                      \
  if (!st) {                                                                \
    int _r = ensure_device(dev);                                            \
    if (_r != CQ_OK) return _r;                                             \
    st = stream_of(dev, s);                                                 \
    if (!st) { set_error("bad stream %d on device %d", s, dev); return CQ_ERR_ARG; } \
  }

extern "C" {

const char* cq_last_error(void) { return g_err; }

int cq_version(int* version) {
  *version = 1;
  return CQ_OK;
}

int cq_device_count(int* count) {
  CQ_CHECK_CUDA(cudaGetDeviceCount(count));
  return CQ_OK;
}

int cq_init_device(int device) { return ensure_device(device); }

int cq_device_props(int device, int* sm_count, int64_t* l2_bytes, int* clock_khz,
                    int64_t* total_mem) {
  cudaDeviceProp prop;
  CQ_CHECK_CUDA(cudaGetDeviceProperties(&prop, device));
  *sm_count = prop.multiProcessorCount;
  *l2_bytes = prop.l2CacheSize;
  int khz = 0;
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, device);
  *clock_khz = khz;
  *total_mem = (int64_t)prop.totalGlobalMem;
  return CQ_OK;
}

int cq_enable_peer(int device, int peer, int* enabled) {
  int can = 0;
  CQ_CHECK_CUDA(cudaDeviceCanAccessPeer(&can, device, peer));
  *enabled = 0;
  if (!can) return CQ_OK;
  CQ_CHECK_CUDA(cudaSetDevice(device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
  } else if (e != cudaSuccess) {
    set_error("cudaDeviceEnablePeerAccess(%d->%d): %s", device, peer, cudaGetErrorString(e));
    return CQ_ERR_CUDA;
  }
  *enabled = 1;
  return CQ_OK;
}

int cq_shutdown(void) {
  for (int i = 0; i < kMaxDevices; ++i) {
    if (!g_dev[i].ready) continue;
    cudaSetDevice(i);
    cudaDeviceSynchronize();
    for (auto& kv : g_pool[i].free_blocks) cudaFree(kv.second);
    g_pool[i].free_blocks.clear();
    free_scratch(i);
    for (int s = 0; s < CQ_NUM_STREAMS; ++s) cudaStreamDestroy(g_dev[i].streams[s]);
    cudaFree(g_dev[i].error_flag);
    g_dev[i] = DeviceState();
  }
  return CQ_OK;
}

// ------------------------------------------------------------------ memory
int cq_malloc(int device, int64_t bytes, void** ptr) {
  CQ_TRY(ensure_device(device));
  CQ_REQUIRE(bytes >= 0, "negative allocation");
  // round to 2 MiB (large) / 256 B (small) so blocks are reusable across runs
  int64_t rounded = bytes <= (1 << 20) ? ((bytes + 255) & ~int64_t(255))
                                       : ((bytes + (2 << 20) - 1) & ~int64_t((2 << 20) - 1));
  if (rounded == 0) rounded = 256;
  std::lock_guard<std::mutex> lk(g_mu);
  Pool& p = g_pool[device];
  auto it = p.free_blocks.find(rounded);
  if (it != p.free_blocks.end()) {
    *ptr = it->second;
    p.free_blocks.erase(it);
  } else {
    CQ_CHECK_CUDA(cudaSetDevice(device));
    cudaError_t e = cudaMalloc(ptr, rounded);
    if (e == cudaErrorMemoryAllocation && !p.free_blocks.empty()) {
      cudaGetLastError();
      for (auto& kv : p.free_blocks) cudaFree(kv.second);
      p.free_blocks.clear();
      e = cudaMalloc(ptr, rounded);
    }
    if (e != cudaSuccess) {
      set_error("cudaMalloc(%lld) on device %d: %s", (long long)rounded, device, cudaGetErrorString(e));
      return CQ_ERR_CUDA;
    }
  }
  p.live[*ptr] = rounded;
  return CQ_OK;
}

int cq_free(int device, void* ptr) {
  if (!ptr) return CQ_OK;
  std::lock_guard<std::mutex> lk(g_mu);
  Pool& p = g_pool[device];
  auto it = p.live.find(ptr);
  CQ_REQUIRE(it != p.live.end(), "cq_free: unknown pointer %p on device %d", ptr, device);
  p.free_blocks.emplace(it->second, ptr);
  p.live.erase(it);
  return CQ_OK;
}

int cq_pool_trim(int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  CQ_CHECK_CUDA(cudaSetDevice(device));
  CQ_CHECK_CUDA(cudaDeviceSynchronize());
  for (auto& kv : g_pool[device].free_blocks) cudaFree(kv.second);
  g_pool[device].free_blocks.clear();
  return CQ_OK;
}

int cq_host_alloc(int64_t bytes, void** ptr) {
  CQ_REQUIRE(bytes > 0 && ptr != nullptr, "cq_host_alloc: bad arguments");
  CQ_CHECK_CUDA(cudaMallocHost(ptr, (size_t)bytes));
  return CQ_OK;
}

int cq_host_free(void* ptr) {
  if (ptr) CQ_CHECK_CUDA(cudaFreeHost(ptr));
  return CQ_OK;
}

int cq_host_register(void* ptr, int64_t bytes) {
  cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterPortable);
  if (e == cudaErrorHostMemoryAlreadyRegistered) {
    cudaGetLastError();
    return CQ_OK;
  }
  if (e != cudaSuccess) {
    set_error("cudaHostRegister: %s", cudaGetErrorString(e));
    return CQ_ERR_CUDA;
  }
  return CQ_OK;
}

int cq_host_unregister(void* ptr) {
  cudaError_t e = cudaHostUnregister(ptr);
  if (e == cudaErrorHostMemoryNotRegistered) {
    cudaGetLastError();
    return CQ_OK;
  }
  if (e != cudaSuccess) {
    set_error("cudaHostUnregister: %s", cudaGetErrorString(e));
    return CQ_ERR_CUDA;
  }
  return CQ_OK;
}

// ------------------------------------------------------------------ copies
int cq_copy_h2d(int device, int stream, void* dst, const void* src, int64_t bytes) {
  CQ_STREAM(device, stream);
  if (bytes == 0) return CQ_OK;
  CQ_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
  return CQ_OK;
}

int cq_copy_d2h(int device, int stream, void* dst, const void* src, int64_t bytes) {
  CQ_STREAM(device, stream);
  if (bytes == 0) return CQ_OK;
  CQ_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
  return CQ_OK;
}

}  // extern "C"

namespace cq {

// Byte offset of global cell `p` inside an allocation box with element strides.
static inline int64_t cell_offset(const cq_box_t& alloc, const int64_t* stride, const int64_t* p) {
  int64_t off = 0;
  for (int k = 0; k < CQ_MAX_DIMS; ++k) off += (p[k] - alloc.lo[k]) * stride[k];
  return off;
}

static inline void dense_strides(const cq_box_t& b, int64_t* s) {
  s[2] = 1;
  s[1] = b.hi[2] - b.lo[2];
  s[0] = s[1] * (b.hi[1] - b.lo[1]);
}

static inline bool box_inside(const cq_box_t& in, const cq_box_t& outer) {
  for (int k = 0; k < CQ_MAX_DIMS; ++k)
    if (in.lo[k] < outer.lo[k] || in.hi[k] > outer.hi[k]) return false;
  return true;
}

// Is the box one contiguous run of the (dense, row-major) allocation?  True
// when every axis after the first non-unit one spans the allocation fully.
static inline bool box_contiguous(const cq_box_t& box, const cq_box_t& alloc) {
  int k = 0;
  while (k < CQ_MAX_DIMS - 1 && box.hi[k] - box.lo[k] == 1) ++k;
  for (int j = k + 1; j < CQ_MAX_DIMS; ++j)
    if (box.hi[j] - box.lo[j] != alloc.hi[j] - alloc.lo[j]) return false;
  return true;
}

// Strided box copy.  Boxes are 3-D with the innermost (contiguous) axis last;
// lower-dimensional buffers pad LEADING axes with [0,1).  Uses one flat copy
// when both sides are contiguous, one 2-D DMA when the rows have a single
// pitch, else one 2-D DMA per axis-0 slab.
static int copy_box_generic(cudaStream_t st, int eb, char* dst, const cq_box_t& dalloc,
                            const int64_t* dstride, const char* src, const cq_box_t& salloc,
                            const int64_t* sstride, const cq_box_t& box, cudaMemcpyKind kind) {
  int64_t n0 = box.hi[0] - box.lo[0], n1 = box.hi[1] - box.lo[1], n2 = box.hi[2] - box.lo[2];
  if (n0 <= 0 || n1 <= 0 || n2 <= 0) return CQ_OK;
  int64_t p[3] = {box.lo[0], box.lo[1], box.lo[2]};
  char* d0 = dst + cell_offset(dalloc, dstride, p) * eb;
  const char* s0 = src + cell_offset(salloc, sstride, p) * eb;
  if (box_contiguous(box, dalloc) && box_contiguous(box, salloc)) {
    size_t bytes = (size_t)(n0 * n1 * n2 * eb);
    cudaError_t e = cudaMemcpyAsync(d0, s0, bytes, kind, st);
    if (e != cudaSuccess) {
      cudaGetLastError();
      cudaPointerAttributes ad = {}, as = {};
      cudaPointerGetAttributes(&ad, d0);
      cudaGetLastError();
      cudaPointerGetAttributes(&as, s0);
      cudaGetLastError();
      int cur = -1;
      cudaGetDevice(&cur);
      set_error("cudaMemcpyAsync(dst=%p type %d dev %d, src=%p type %d dev %d, %zu B, kind %d, cur dev %d): %s", d0,
                (int)ad.type, ad.device, s0, (int)as.type, as.device, bytes, (int)kind, cur, cudaGetErrorString(e));
      return CQ_ERR_CUDA;
    }
    return CQ_OK;
  }
  if (n0 == 1) {
    CQ_CHECK_CUDA(cudaMemcpy2DAsync(d0, dstride[1] * eb, s0, sstride[1] * eb, n2 * eb, n1, kind, st));
    return CQ_OK;
  }
  if (n1 == 1) {
    CQ_CHECK_CUDA(cudaMemcpy2DAsync(d0, dstride[0] * eb, s0, sstride[0] * eb, n2 * eb, n0, kind, st));
    return CQ_OK;
  }
  if (n1 == dalloc.hi[1] - dalloc.lo[1] && n1 == salloc.hi[1] - salloc.lo[1]) {
    CQ_CHECK_CUDA(cudaMemcpy2DAsync(d0, dstride[1] * eb, s0, sstride[1] * eb, n2 * eb, n0 * n1,
                                    kind, st));
    return CQ_OK;
  }
  for (int64_t i = 0; i < n0; ++i) {
    p[0] = box.lo[0] + i;
    CQ_CHECK_CUDA(cudaMemcpy2DAsync(dst + cell_offset(dalloc, dstride, p) * eb, dstride[1] * eb,
                                    src + cell_offset(salloc, sstride, p) * eb, sstride[1] * eb,
                                    n2 * eb, n1, kind, st));
  }
  return CQ_OK;
}

}  // namespace cq

extern "C" {

int cq_copy_box(int device, int stream, int elem_bytes, const cq_view_t* dst, int dst_device,
                const cq_view_t* src, int src_device, const cq_box_t* box) {
  CQ_STREAM(device, stream);
  CQ_REQUIRE(box_inside(*box, dst->alloc) && box_inside(*box, src->alloc),
             "cq_copy_box: box outside an allocation");
  cudaMemcpyKind kind = cudaMemcpyDeviceToDevice;
  (void)dst_device;
  (void)src_device;  // unified addressing: peer copies route over NVLink
  return copy_box_generic(st, elem_bytes, (char*)dst->ptr, dst->alloc, dst->stride,
                          (const char*)src->ptr, src->alloc, src->stride, *box, kind);
}

int cq_copy_box_h2d(int device, int stream, int elem_bytes, const cq_view_t* dst,
                    const void* host, const cq_box_t* host_alloc, const cq_box_t* box) {
  CQ_STREAM(device, stream);
  CQ_REQUIRE(box_inside(*box, dst->alloc) && box_inside(*box, *host_alloc),
             "cq_copy_box_h2d: box outside an allocation");
  int64_t hs[3];
  dense_strides(*host_alloc, hs);
  return copy_box_generic(st, elem_bytes, (char*)dst->ptr, dst->alloc, dst->stride,
                          (const char*)host, *host_alloc, hs, *box, cudaMemcpyHostToDevice);
}

int cq_copy_box_d2h(int device, int stream, int elem_bytes, void* host,
                    const cq_box_t* host_alloc, const cq_view_t* src, const cq_box_t* box) {
  CQ_STREAM(device, stream);
  CQ_REQUIRE(box_inside(*box, src->alloc) && box_inside(*box, *host_alloc),
             "cq_copy_box_d2h: box outside an allocation");
  int64_t hs[3];
  dense_strides(*host_alloc, hs);
  return copy_box_generic(st, elem_bytes, (char*)host, *host_alloc, hs, (const char*)src->ptr,
                          src->alloc, src->stride, *box, cudaMemcpyDeviceToHost);
}

int cq_pack_box(int device, int stream, int elem_bytes, void* dense, const cq_view_t* src,
                const cq_box_t* box) {
  CQ_STREAM(device, stream);
  CQ_REQUIRE(box_inside(*box, src->alloc), "cq_pack_box: box outside the allocation");
  int64_t ds[3];
  dense_strides(*box, ds);
  return copy_box_generic(st, elem_bytes, (char*)dense, *box, ds, (const char*)src->ptr,
                          src->alloc, src->stride, *box, cudaMemcpyDeviceToDevice);
}

int cq_unpack_box(int device, int stream, int elem_bytes, const cq_view_t* dst,
                  const void* dense, const cq_box_t* box) {
  CQ_STREAM(device, stream);
  CQ_REQUIRE(box_inside(*box, dst->alloc), "cq_unpack_box: box outside the allocation");
  int64_t ds[3];
  dense_strides(*box, ds);
  return copy_box_generic(st, elem_bytes, (char*)dst->ptr, dst->alloc, dst->stride,
                          (const char*)dense, *box, ds, *box, cudaMemcpyDeviceToDevice);
}

// ------------------------------------------------------------------ events
int cq_event_create(int device, int timing, uint64_t* event) {
  CQ_TRY(ensure_device(device));
  CQ_CHECK_CUDA(cudaSetDevice(device));
  cudaEvent_t e;
  CQ_CHECK_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
  *event = (uint64_t)(uintptr_t)e;
  return CQ_OK;
}

int cq_event_destroy(uint64_t event) {
  CQ_CHECK_CUDA(cudaEventDestroy((cudaEvent_t)(uintptr_t)event));
  return CQ_OK;
}

int cq_event_record(uint64_t event, int device, int stream) {
  CQ_STREAM(device, stream);
  CQ_CHECK_CUDA(cudaEventRecord((cudaEvent_t)(uintptr_t)event, st));
  return CQ_OK;
}

int cq_event_record_timed(uint64_t event, int device, int stream) {
  CQ_STREAM(device, stream);
  cudaStreamCaptureStatus cs;
  CQ_CHECK_CUDA(cudaStreamIsCapturing(st, &cs));
  if (cs == cudaStreamCaptureStatusActive)
    CQ_CHECK_CUDA(cudaEventRecordWithFlags((cudaEvent_t)(uintptr_t)event, st, cudaEventRecordExternal));
  else
    CQ_CHECK_CUDA(cudaEventRecord((cudaEvent_t)(uintptr_t)event, st));
  return CQ_OK;
}

int cq_stream_wait_event(int device, int stream, uint64_t event) {
  CQ_STREAM(device, stream);
  CQ_CHECK_CUDA(cudaStreamWaitEvent(st, (cudaEvent_t)(uintptr_t)event, 0));
  return CQ_OK;
}

int cq_event_synchronize(uint64_t event) {
  CQ_CHECK_CUDA(cudaEventSynchronize((cudaEvent_t)(uintptr_t)event));
  return CQ_OK;
}

int cq_event_elapsed_ms(uint64_t start, uint64_t stop, float* ms) {
  CQ_CHECK_CUDA(cudaEventElapsedTime(ms, (cudaEvent_t)(uintptr_t)start, (cudaEvent_t)(uintptr_t)stop));
  return CQ_OK;
}

int cq_stream_synchronize(int device, int stream) {
  CQ_STREAM(device, stream);
  CQ_CHECK_CUDA(cudaStreamSynchronize(st));
  return CQ_OK;
}

int cq_device_synchronize(int device) {
  CQ_CHECK_CUDA(cudaSetDevice(device));
  CQ_CHECK_CUDA(cudaDeviceSynchronize());
  return CQ_OK;
}

// ------------------------------------------------------------ graph capture
// Fork: the compute stream starts a (relaxed-mode) capture and the boundary
// and comm streams join it through an event; join: both record an event the
// compute stream waits on before the capture ends.
int cq_graph_begin(int device) {
  CQ_STREAM(device, CQ_STREAM_COMPUTE);
  CQ_CHECK_CUDA(cudaSetDevice(device));
  CQ_CHECK_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
  cudaEvent_t fork;
  CQ_CHECK_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  CQ_CHECK_CUDA(cudaEventRecord(fork, st));
  for (int s = 1; s < CQ_NUM_STREAMS; ++s) CQ_CHECK_CUDA(cudaStreamWaitEvent(stream_of(device, s), fork, 0));
  CQ_CHECK_CUDA(cudaEventDestroy(fork));
  return CQ_OK;
}

int cq_graph_end(int device, uint64_t* graph) {
  CQ_STREAM(device, CQ_STREAM_COMPUTE);
  CQ_CHECK_CUDA(cudaSetDevice(device));
  for (int s = 1; s < CQ_NUM_STREAMS; ++s) {
    cudaEvent_t join;
    CQ_CHECK_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    CQ_CHECK_CUDA(cudaEventRecord(join, stream_of(device, s)));
    CQ_CHECK_CUDA(cudaStreamWaitEvent(st, join, 0));
    CQ_CHECK_CUDA(cudaEventDestroy(join));
  }
  cudaGraph_t g = nullptr;
  CQ_CHECK_CUDA(cudaStreamEndCapture(st, &g));
  cudaGraphExec_t exec = nullptr;
  cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    set_error("cudaGraphInstantiate: %s", cudaGetErrorString(e));
    return CQ_ERR_CUDA;
  }
  *graph = (uint64_t)(uintptr_t)exec;
  return CQ_OK;
}

int cq_graph_launch(uint64_t graph, int device) {
  CQ_STREAM(device, CQ_STREAM_COMPUTE);
  CQ_CHECK_CUDA(cudaGraphLaunch((cudaGraphExec_t)(uintptr_t)graph, st));
  return CQ_OK;
}

int cq_graph_destroy(uint64_t graph) {
  CQ_CHECK_CUDA(cudaGraphExecDestroy((cudaGraphExec_t)(uintptr_t)graph));
  return CQ_OK;
}

// -------------------------------------------------------------------- NCCL
static ncclComm_t g_comm = nullptr;
static int g_comm_device = -1;

#define CQ_CHECK_NCCL(expr)                                                         \
  do {                                                                              \
    ncclResult_t _r = (expr);                                                       \
    if (_r != ncclSuccess) {                                                        \
      set_error("%s:%d: %s: %s", __FILE__, __LINE__, #expr, ncclGetErrorString(_r)); \
      return CQ_ERR_NCCL;                                                           \
    }                                                                               \
  } while (0)

int cq_nccl_unique_id(unsigned char id_out[128]) {
  ncclUniqueId id;
  CQ_CHECK_NCCL(ncclGetUniqueId(&id));
  memcpy(id_out, id.internal, 128);
  return CQ_OK;
}

int cq_nccl_init(int device, int nranks, int rank, const unsigned char id[128]) {
  CQ_TRY(ensure_device(device));
  CQ_CHECK_CUDA(cudaSetDevice(device));
  ncclUniqueId uid;
  memcpy(uid.internal, id, 128);
  CQ_CHECK_NCCL(ncclCommInitRank(&g_comm, nranks, uid, rank));
  g_comm_device = device;
  return CQ_OK;
}

int cq_nccl_group_start(void) {
  CQ_CHECK_NCCL(ncclGroupStart());
  return CQ_OK;
}

int cq_nccl_group_end(void) {
  CQ_CHECK_NCCL(ncclGroupEnd());
  return CQ_OK;
}

int cq_nccl_send(int device, int stream, const void* buf, int64_t bytes, int peer) {
  CQ_STREAM(device, stream);
  CQ_REQUIRE(g_comm && device == g_comm_device, "NCCL not initialised for device %d", device);
  CQ_CHECK_NCCL(ncclSend(buf, (size_t)bytes, ncclChar, peer, g_comm, st));
  return CQ_OK;
}

int cq_nccl_recv(int device, int stream, void* buf, int64_t bytes, int peer) {
  CQ_STREAM(device, stream);
  CQ_REQUIRE(g_comm && device == g_comm_device, "NCCL not initialised for device %d", device);
  CQ_CHECK_NCCL(ncclRecv(buf, (size_t)bytes, ncclChar, peer, g_comm, st));
  return CQ_OK;
}

int cq_nccl_allgather(int device, int stream, const void* send, void* recv, int64_t bytes_per_rank) {
  CQ_STREAM(device, stream);
  CQ_REQUIRE(g_comm && device == g_comm_device, "NCCL not initialised for device %d", device);
  CQ_CHECK_NCCL(ncclAllGather(send, recv, (size_t)bytes_per_rank, ncclChar, g_comm, st));
  return CQ_OK;
}

int cq_nccl_bcast(int device, int stream, void* buf, int64_t bytes, int root) {
  CQ_STREAM(device, stream);
  CQ_REQUIRE(g_comm && device == g_comm_device, "NCCL not initialised for device %d", device);
  CQ_CHECK_NCCL(ncclBroadcast(buf, buf, (size_t)bytes, ncclChar, root, g_comm, st));
  return CQ_OK;
}

// ------------------------------------------------------------ CUDA IPC
int cq_ipc_handle(const void* ptr, unsigned char handle_out[64]) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  CQ_CHECK_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(ptr)));
  memcpy(handle_out, &h, sizeof(h));
  return CQ_OK;
}

int cq_ipc_open(int device, const unsigned char handle[64], void** ptr) {
  CQ_TRY(ensure_device(device));
  CQ_CHECK_CUDA(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  CQ_CHECK_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return CQ_OK;
}

int cq_ipc_close(int device, void* ptr) {
  CQ_CHECK_CUDA(cudaSetDevice(device));
  CQ_CHECK_CUDA(cudaIpcCloseMemHandle(ptr));
  return CQ_OK;
}

int cq_nccl_destroy(void) {
  if (g_comm) {
    ncclCommDestroy(g_comm);
    g_comm = nullptr;
    g_comm_device = -1;
  }
  return CQ_OK;
}

}  // extern "C"
