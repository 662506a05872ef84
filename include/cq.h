/*
 * libcq -- C-ABI of the B200-native executor for the Celerity/SYnergy-style
 * data-parallel path of arXiv 2505.06022.
 *
 * The reference (clusterq) has no native boundary: its executor is the Python
 * simulator run(plan) (pkg/src/clusterq/simulator.py:101-224).  Each entry
 * point below replaces one data-plane operation of that simulator; the
 * citation names the reference code it stands in for.  The Python executor
 * (paper_2505_06022_b200/executor.py) is the only caller, through ctypes.
 *
 * Conventions
 *   - every function returns int: CQ_OK (0) or a CQ_ERR_* code; the message
 *     is available from cq_last_error() (thread-local);
 *   - plain pointers and sizes only: device pointers come from cq_malloc,
 *     host pointers are caller-owned (pin with cq_host_register);
 *   - all work is asynchronous on the stream named by (device, stream) with
 *     stream in {CQ_STREAM_COMPUTE, CQ_STREAM_BOUNDARY, CQ_STREAM_COMM,
 *     CQ_STREAM_LANE0 .. CQ_STREAM_LANE0 + CQ_NUM_LANES - 1};
 *   - element kinds: CQ_F64 / CQ_F32 / CQ_I64.
 *   - one process may own several devices; multi-process runs use NCCL
 *     (cq_nccl_*), one rank per GPU.
 */
#ifndef CQ_H
#define CQ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  CQ_OK = 0,
  CQ_ERR_CUDA = 1,
  CQ_ERR_NCCL = 2,
  CQ_ERR_NVML = 3,
  CQ_ERR_ARG = 4,
  CQ_ERR_PERMISSION = 5,
  CQ_ERR_UNSUPPORTED = 6,
  CQ_ERR_EVAL = 7,     /* integer division by zero  -> EvalError            */
  CQ_ERR_MAPPER = 8,   /* read outside mapped region -> MapperViolationError */
  CQ_ERR_P2P = 9       /* a peer's halo signal did not arrive in time (device flag) */
};

enum { CQ_F64 = 0, CQ_F32 = 1, CQ_I64 = 2 };
/* Lanes: extra default-priority compute streams, so the executes of several
 * plan nodes sharing one device (independent allocations) run concurrently. */
enum {
  CQ_STREAM_COMPUTE = 0,
  CQ_STREAM_BOUNDARY = 1,
  CQ_STREAM_COMM = 2,
  CQ_STREAM_LANE0 = 3,
  CQ_NUM_LANES = 8,
  CQ_NUM_STREAMS = 11
};

#define CQ_MAX_DIMS 3

/* A box of cells [lo, hi) in global buffer coordinates (reference Box,
 * region.py:18-101).  Always 3-D with the innermost (contiguous) axis last: a
 * d-dimensional buffer occupies the LAST d axes and leading axes are [0, 1). */
typedef struct {
  int64_t lo[CQ_MAX_DIMS];
  int64_t hi[CQ_MAX_DIMS];
} cq_box_t;

/* A node-local allocation holding the cells of `alloc` (the bounding box of
 * everything the node touches), row-major; stride[] in elements.  Global
 * cell p lives at ptr + sum_k (p[k] - alloc.lo[k]) * stride[k]. */
typedef struct {
  void* ptr;
  cq_box_t alloc;
  int64_t stride[CQ_MAX_DIMS];
} cq_view_t;

/* ------------------------------------------------------------------ runtime */
const char* cq_last_error(void);
int cq_version(int* version);
int cq_device_count(int* count);
/* Create streams and the event pool of `device` (idempotent). */
int cq_init_device(int device);
/* sm count, l2 bytes, max sm clock kHz, total memory bytes */
int cq_device_props(int device, int* sm_count, int64_t* l2_bytes, int* clock_khz,
                    int64_t* total_mem);
int cq_enable_peer(int device, int peer, int* enabled);
int cq_shutdown(void);

/* Pooled device memory (caching allocator; blocks are reused by size). */
int cq_malloc(int device, int64_t bytes, void** ptr);
int cq_free(int device, void* ptr);
int cq_pool_trim(int device);
int cq_host_register(void* ptr, int64_t bytes);
int cq_host_unregister(void* ptr);
/* Page-locked host memory owned by libcq (small staging buffers). */
int cq_host_alloc(int64_t bytes, void** ptr);
int cq_host_free(void* ptr);

/* Copies -- the Push/AwaitPush payload move (simulator.py:166-193) and the
 * final gather (simulator.py:210-222). Box copies are 2-D/3-D strided DMA
 * between views on the same or a peer device of this process. */
int cq_copy_h2d(int device, int stream, void* dst, const void* src, int64_t bytes);
int cq_copy_d2h(int device, int stream, void* dst, const void* src, int64_t bytes);
int cq_copy_box(int device, int stream, int elem_bytes, const cq_view_t* dst, int dst_device,
                const cq_view_t* src, int src_device, const cq_box_t* box);
int cq_copy_box_h2d(int device, int stream, int elem_bytes, const cq_view_t* dst,
                    const void* host, const cq_box_t* host_alloc, const cq_box_t* box);
int cq_copy_box_d2h(int device, int stream, int elem_bytes, void* host,
                    const cq_box_t* host_alloc, const cq_view_t* src, const cq_box_t* box);
/* Pack a box of a view into / out of a dense staging buffer (for NCCL). */
int cq_pack_box(int device, int stream, int elem_bytes, void* dense, const cq_view_t* src,
                const cq_box_t* box);
int cq_unpack_box(int device, int stream, int elem_bytes, const cq_view_t* dst,
                  const void* dense, const cq_box_t* box);

/* Events and stream ordering (command dependencies, scheduler.py:263-348). */
/* timing = 0 creates a cudaEventDisableTiming event (cheaper; ordering only). */
int cq_event_create(int device, int timing, uint64_t* event);
int cq_event_destroy(uint64_t event);
int cq_event_record(uint64_t event, int device, int stream);
/* A timestamp that survives graph capture: while `stream` is being captured
 * it becomes an event-record node (re-recorded on every replay, so the
 * per-launch times of the replayed graph can be read back); otherwise it is
 * cq_event_record.  Trace-only: never waited on. */
int cq_event_record_timed(uint64_t event, int device, int stream);
int cq_stream_wait_event(int device, int stream, uint64_t event);
int cq_event_synchronize(uint64_t event);
int cq_event_elapsed_ms(uint64_t start, uint64_t stop, float* ms);
int cq_stream_synchronize(int device, int stream);
int cq_device_synchronize(int device);

/* CUDA-graph capture of everything issued on the three streams of `device`
 * between begin and end (kernels, copies, NCCL groups, event edges); the
 * executable graph replays the whole plan with one launch. */
int cq_graph_begin(int device);
int cq_graph_end(int device, uint64_t* graph);
int cq_graph_launch(uint64_t graph, int device);
int cq_graph_destroy(uint64_t graph);

/* ------------------------------------------------------------------- NCCL */
int cq_nccl_unique_id(unsigned char id_out[128]);
int cq_nccl_init(int device, int nranks, int rank, const unsigned char id[128]);
int cq_nccl_group_start(void);
int cq_nccl_group_end(void);
int cq_nccl_send(int device, int stream, const void* buf, int64_t bytes, int peer);
int cq_nccl_recv(int device, int stream, void* buf, int64_t bytes, int peer);
int cq_nccl_allgather(int device, int stream, const void* send, void* recv, int64_t bytes_per_rank);
/* In-place broadcast of `bytes` at `buf` from rank `root` (ncclBroadcast): one
 * source node's region pushed to every other node (SURVEY §8b cq_bcast). */
int cq_nccl_bcast(int device, int stream, void* buf, int64_t bytes, int root);
int cq_nccl_destroy(void);

/* ------------------------------------------ peer memory (CUDA IPC, NVLink)
 * The temporally blocked wave's halo rows go straight into the neighbouring
 * rank's allocations (copy-engine writes through IPC-opened pointers) instead
 * of a per-pass NCCL exchange; device-side counters order the passes. */
/* IPC handle (64 bytes) of an allocation's base pointer (cq_malloc blocks). */
int cq_ipc_handle(const void* ptr, unsigned char handle_out[64]);
/* Open a peer process's allocation on `device`; *ptr is valid for copies and
 * device stores until cq_ipc_close. */
int cq_ipc_open(int device, const unsigned char handle[64], void** ptr);
int cq_ipc_close(int device, void* ptr);
/* Block `stream` until every non-null `slot_k` (a local word written by a
 * peer) holds a value >= *count (a local word); after `timeout_ns` the wait
 * gives up and sets the device error flag (CQ_ERR_P2P) instead of hanging. */
int cq_p2p_wait(int device, int stream, const uint64_t* slot0, const uint64_t* slot1, const uint64_t* count,
                int64_t timeout_ns);
/* *count += 1, then store the new value (release, system scope) to every
 * non-null peer word. */
int cq_p2p_signal(int device, int stream, uint64_t* count, uint64_t* peer0, uint64_t* peer1);

/* ----------------------------------------------------------------- kernels */
/* Host-initialised contents of node 0 (BufferInit.materialize, model.py:63-74):
 * mode 0 zeros, 1 iota (row-major index within `extent`), 2 constant. */
int cq_fill(int device, int stream, int kind, const cq_view_t* dst, const cq_box_t* box,
            const cq_box_t* extent, int mode, double value, int64_t ivalue);

/* z[i] = alpha * x[i] + y[i] with one rounding per operator (the bundled
 * saxpy scenario, scenarios/saxpy.json:15, evaluated as kernel.py:291-331).
 * n contiguous cells; kind selects f64 / f32 / wrapping i64. */
int cq_saxpy(int device, int stream, int kind, double alpha, int64_t ialpha, const void* x,
             const void* y, void* z, int64_t n);

/* One leapfrog step of the 2-D 5-point wave body over `box`:
 *   out = ((k2*u) - upr) + (c * ((((uN + uS) + uW) + uE) - (k4*u)))
 * reads of u clamped to `extent` (model.py:442-446); out may alias upr. */
int cq_wave5(int device, int stream, int kind, const cq_view_t* u, const cq_view_t* upr,
             const cq_view_t* out, const cq_box_t* box, const cq_box_t* extent, double c,
             double k2, double k4);
/* KL (4 or 8) wave steps in one HBM pass (temporal blocking): from u = X(t)
 * and upr = X(t-1), readable on rows [in_lo, in_hi), write X(t+KL) to
 * out_last and X(t+KL-1) to out_prev on rows [out_lo, out_hi) x all columns.
 * Bit-identical to KL cq_wave5 launches (same per-cell tree and rounding).
 * kind f32 / f64, whole 16-byte aligned rows, outputs distinct from inputs, k2 = 2, k4 = 4, and
 * [out_lo, out_hi) inside [in_lo + KL, in_hi - KL) except at the borders
 * 0 and H (which clamp like the DSL). */
int cq_wave5_fused(int device, int stream, int kind, int levels, const cq_view_t* u, const cq_view_t* upr,
                   const cq_view_t* out_last, const cq_view_t* out_prev, int64_t in_lo, int64_t in_hi,
                   int64_t out_lo, int64_t out_hi, const cq_box_t* extent, double c, double k2, double k4);
/* The same pass with a magnitude bound: amax_in (device float, or NULL)
 * bounds |X(t)|, |X(t-1)| over the rows this launch reads; when it is below
 * 2^124 / (3 + 8|c|)^levels the interior blocks use an FMA form of the body
 * that is bit-identical while nothing overflows (7 instead of 9 FP
 * operations per cell).  amax_out (device float, or NULL) receives, by
 * atomic max, max |value| over the rows written -- the next pass's amax_in.
 * cq_wave5_fused == this with both NULL. */
int cq_wave5_fused_bounded(int device, int stream, int kind, int levels, const cq_view_t* u, const cq_view_t* upr,
                           const cq_view_t* out_last, const cq_view_t* out_prev, int64_t in_lo, int64_t in_hi,
                           int64_t out_lo, int64_t out_hi, const cq_box_t* extent, double c, double k2, double k4,
                           const float* amax_in, float* amax_out);
/* A peer rank's output allocations (CUDA IPC pointers) that also receive
 * the rows [row_lo, row_hi) a fused pass writes: X(t+KL) rows to `last`, X(t+KL-1)
 * rows to `prev`; the cell (r, c) lives at base + (r - row0) * stride + (c - col0). */
typedef struct {
  void* last;
  void* prev;
  int64_t row0, col0, stride;
  int64_t row_lo, row_hi;
} cq_mirror_t;

/* In-pass ordering with the neighbouring ranks (executor._PeerHalo): the
 * blocks whose pieces read halo rows / store mirrored rows first wait until
 * every non-null local `slot` (written by a neighbour) >= *count, and the last
 * of them to finish increments *count and stores it (release, system scope)
 * to every non-null `peer_slot`, after raising every non-null `peer_amax` with
 * its rows' max |x|.  `done` is a local zeroed counter. */
typedef struct {
  const uint64_t* slot[2];
  uint64_t* count;
  uint32_t* done;
  uint64_t* peer_slot[2];
  float* peer_amax[2];    /* the neighbours' amax_out words: edge blocks raise them too */
  int64_t timeout_ns;
} cq_peer_sync_t;

/* cq_wave5_fused_bounded whose FMA form (amax_in) covers only pieces reading
 * rows inside [fast_lo, fast_hi) -- e.g. not a neighbour's halo rows, which
 * the local bound does not cover; the others keep the exact form -- and whose
 * output rows inside a mirror's range are also stored to that peer (up to 2;
 * the storing blocks end with a system-scope fence). */
int cq_wave5_fused_ex(int device, int stream, int kind, int levels, const cq_view_t* u, const cq_view_t* upr,
                      const cq_view_t* out_last, const cq_view_t* out_prev, int64_t in_lo, int64_t in_hi,
                      int64_t out_lo, int64_t out_hi, const cq_box_t* extent, double c, double k2, double k4,
                      const float* amax_in, float* amax_out, int64_t fast_lo, int64_t fast_hi,
                      const cq_mirror_t* mirrors, int n_mirrors, const cq_peer_sync_t* sync);

/* Geometry of one fused pass over `rows` output rows of a W-column grid:
 * out = {rows per warp piece, blocks, warps, cells computed per level by
 * the launched warps (halo columns / rows included)}.  Host-side query for
 * the roofline's recompute share (bench.py); launches nothing. */
int cq_wave5_fused_geometry(int device, int kind, int levels, int64_t rows, int64_t W, int64_t out[4]);

/* Device interpreter for arbitrary task bodies (eval_kernel, kernel.py:291-331
 * with ReadView clamping + mapper check, model.py:442-453). */
#define CQ_EXPR_MAX_CODE 192
#define CQ_EXPR_MAX_CONST 64
#define CQ_EXPR_MAX_SLOTS 24
#define CQ_EXPR_MAX_VIEWS 8
#define CQ_EXPR_MAX_OUT 4
#define CQ_EXPR_MAX_CHECK_BOXES 8
typedef struct {
  int32_t kind;                 /* CQ_F64 / CQ_F32 / CQ_I64 */
  int32_t dims;                 /* kernel dimensionality */
  cq_box_t box;                 /* cells to evaluate (global coordinates) */
  int32_t n_out;
  int32_t out_code_begin[CQ_EXPR_MAX_OUT];
  int32_t out_code_end[CQ_EXPR_MAX_OUT];
  cq_view_t out[CQ_EXPR_MAX_OUT];
  int32_t n_code;
  int16_t code_op[CQ_EXPR_MAX_CODE];
  int16_t code_arg[CQ_EXPR_MAX_CODE];
  int32_t n_const;
  int64_t consts[CQ_EXPR_MAX_CONST]; /* bit patterns (double / int64) */
  int32_t n_slots;
  int32_t slot_view[CQ_EXPR_MAX_SLOTS];
  int32_t slot_off[CQ_EXPR_MAX_SLOTS][CQ_MAX_DIMS];
  int32_t n_views;
  cq_view_t views[CQ_EXPR_MAX_VIEWS];
  cq_box_t view_extent[CQ_EXPR_MAX_VIEWS];
  int32_t view_dims[CQ_EXPR_MAX_VIEWS];
  int32_t view_n_check[CQ_EXPR_MAX_VIEWS];   /* 0: no mapper check needed */
  cq_box_t view_check[CQ_EXPR_MAX_VIEWS][CQ_EXPR_MAX_CHECK_BOXES];
} cq_expr_t;
int cq_expr_eval(int device, int stream, const cq_expr_t* expr);
/* DSL -> CUDA JIT: compile straight-line CUDA for a body with NVRTC (sm_100a)
 * and launch it on the same cq_expr_t block (bit-identical to cq_expr_eval).
 * `headers` are in-memory include files (cq.h itself). */
int cq_jit_compile(const char* source, const char* kernel_name, int n_headers, const char** header_src,
                   const char** header_names, uint64_t* handle);
int cq_jit_launch(uint64_t handle, int device, int stream, const cq_expr_t* expr);
/* Sticky per-device error flag written by cq_expr_eval: code 0 / CQ_ERR_EVAL /
 * CQ_ERR_MAPPER with the first failing cell (row-major minimum). */
int cq_error_flag(int device, int* code, int64_t point[CQ_MAX_DIMS], int clear);
/* The same flag copied asynchronously on `stream` into 32 bytes of page-locked
 * host memory (cq_host_alloc): {key, point[3]}, key ~0 = no error, else the
 * low 4 bits are the code.  Lets a pipelined caller check a run without a
 * blocking read that would queue behind other runs' transfers. */
int cq_error_flag_async(int device, int stream, void* host32);

/* All-pairs N-body kick: for i in [i_lo, i_hi): v_i += dt * sum_j m_j d_ij /
 * (|d_ij|^2 + eps2)^(3/2), d_ij = p_j - p_i; pos holds all n bodies (float4
 * x,y,z,m, indexed globally); vel_in / vel point at body i_lo (vel may alias
 * vel_in).  The j order is fixed and independent of i_lo / the GPU count. */
int cq_nbody_kick(int device, int stream, const float* pos, int64_t n, const float* vel_in,
                  float* vel, int64_t i_lo, int64_t i_hi, float eps2, float dt);
/* The kick in pieces, so the j range already on the GPU is computed while
 * the rest is still arriving (an 'all' mapper's all-gather, reference
 * model.py:197-206): j is cut into cq_nbody_jcols() fixed columns, column c
 * = bodies [floor(n c / C), floor(n (c+1) / C)).  kick_partial writes the
 * per-body partial sums of columns [col_lo, col_hi) into part
 * ([C][i_hi - i_lo][3] floats); kick_finalize adds the C columns in column
 * order to vel_in.  Any split of the columns gives cq_nbody_kick's bits. */
int cq_nbody_jcols(int* cols);
int cq_nbody_kick_partial(int device, int stream, const float* pos, int64_t n, float* part, int64_t i_lo,
                          int64_t i_hi, float eps2, int col_lo, int col_hi);
int cq_nbody_kick_finalize(int device, int stream, const float* part, const float* vel_in, float* vel,
                           int64_t count, float dt);
/* p_i.xyz += dt * v_i.xyz for `count` bodies (p may alias p_in). */
int cq_nbody_drift(int device, int stream, const float* p_in, const float* v, float* p,
                   int64_t count, float dt);

/* C[m x n] = A[m x k] . B[k x n], row-major with leading dimensions in
 * elements. variant 0 = FFMA (SIMT fp32), 1 = 3xTF32 on tcgen05. */
enum { CQ_SGEMM_FFMA = 0, CQ_SGEMM_3XTF32 = 1 };
int cq_sgemm(int device, int stream, int variant, const float* a, int64_t lda, const float* b,
             int64_t ldb, float* c, int64_t ldc, int64_t m, int64_t n, int64_t k);

/* ---------------------------------------------------------------- planner */
/* Native generate_commands (reference scheduler.py:224-369, region algebra
 * region.py:113-170): host-only, no GPU needed.  `program` / `*out` use the
 * int64 wire format documented in csrc/cq_plan.cpp; free *out with
 * cq_plan_free. */
int cq_plan_generate(const int64_t* program, int64_t length, int node_count, int64_t** out,
                     int64_t* out_length);
int cq_plan_free(int64_t* out);

/* ------------------------------------------------------------------- NVML */
int cq_nvml_init(void);
int cq_nvml_energy_mj(int device, uint64_t* mj);
int cq_nvml_power_mw(int device, unsigned int* mw);
int cq_nvml_sm_clock_mhz(int device, unsigned int* current, unsigned int* max);
int cq_nvml_throttle_reasons(int device, unsigned long long* reasons);
int cq_nvml_supported_sm_clocks(int device, unsigned int* mhz, int* count);
/* Clock locking changes shared hardware state: refused with
 * CQ_ERR_PERMISSION unless CQ_ALLOW_CLOCK_LOCK=1 is set in the environment. */
int cq_nvml_lock_sm_clock(int device, unsigned int mhz);
int cq_nvml_reset_sm_clock(int device);

#ifdef __cplusplus
}
#endif

#endif /* CQ_H */
